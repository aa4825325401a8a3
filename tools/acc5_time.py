import sys, time, json
sys.path.insert(0, '/root/repo')
import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import engine as E
field = pam.box_field_2d()
part = pam.make_partition(field.mesh, 1, 1)
cfg = pam.AdaptiveConfig(k_top=204, m_max=1836, eta=0.5, m_q=3, max_rounds=4,
                         elastic=pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=4000),
                         offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
for form, kern in (("gram", "auto"), ("residual", "block"), ("residual", "pair")):
    with E.options(cd_form=form, cd_kernel=kern):
        t = time.perf_counter()
        sur, rep = pam.fit_parallel(field, part, cfg, pam.DictionarySpec(sigma=0.031))
        print(json.dumps({"form": form, "kernel": kern, "s": time.perf_counter() - t,
                          "cd": rep.device["kernel_seconds"]["cd"]}), flush=True)
