"""One C5 fit batch (Gram-form CD) for profiling: python tools/c5_probe.py M [n_sub]."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2605_16564_b200 as pam
    from paper_2605_16564_b200 import workloads

    M = int(sys.argv[1])
    n_sub = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    p = workloads.config5_device(M=M, n_sub=n_sub)
    t = time.perf_counter()
    res = pam.fit_subdomains(p)
    print(f"M={M} n_sub={n_sub} fit {time.perf_counter() - t:.3f}s kernel_s {res.kernel_seconds}", flush=True)


if __name__ == "__main__":
    main()
