"""CPU tests of the host-side API mirror (validation, partition logic, batch
bookkeeping, persistence) — everything that does not launch a kernel."""

import io

import numpy as np
import pytest

import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import engine
from paper_2605_16564_b200.partition import _LazyChecksumMeta


def test_config_validation():
    with pytest.raises(ValueError):
        pam.AdaptiveConfig(k_top=0)
    with pytest.raises(ValueError):
        pam.AdaptiveConfig(eta=1.0)
    with pytest.raises(ValueError):
        pam.AdaptiveConfig(m_q=2).offsets_for_dim(1)
    pam.AdaptiveConfig(m_q=2, offsets=((0.0,), (0.25,)))
    with pytest.raises(ValueError):
        pam.AdaptiveConfig(offsets=((0.0,),))
    with pytest.raises(ValueError):
        pam.ElasticNetConfig(lam1=-1.0)
    with pytest.raises(ValueError):
        pam.ElasticNetConfig(tol=0.0)
    with pytest.raises(ValueError):
        pam.DictionarySpec(sigma=0.0)
    with pytest.raises(ValueError, match="entry 1"):
        pam.RbfDictionary(centers=np.array([[0.0], [1.0]]), widths=np.array([0.1, -0.1]))


def test_soft_threshold():
    assert pam.soft_threshold(0.5, 1.0) == 0.0
    assert pam.soft_threshold(2.0, 1.0) == 1.0
    assert pam.soft_threshold(-2.0, 0.5) == -1.5
    with pytest.raises(ValueError):
        pam.soft_threshold(1.0, -0.1)


def test_mesh_and_partition_reference_cases():
    mesh = pam.build_mesh(2, (32, 32), ((0, 1), (0, 1)))
    assert mesh.n_cells == 1024 and mesh.cell_size == (1 / 32, 1 / 32)
    part = pam.make_partition(mesh, 2, 2)
    np.testing.assert_array_equal(np.bincount(part.cell_to_subdomain), [256] * 4)
    part = pam.make_partition(mesh, 2, 1)
    assert part.boxes[0].hi[0] == 0.5 and part.boxes[0].open_hi == (True, False)
    with pytest.raises(ValueError, match="px=3"):
        pam.make_partition(mesh, 3, 2)
    with pytest.raises(ValueError, match="pz must be 1"):
        pam.make_partition(mesh, 2, 2, 2)
    m1 = pam.build_mesh(1, 16, (0.0, 1.0))
    with pytest.raises(ValueError, match="py must be 1"):
        pam.make_partition(m1, 2, 2)
    mesh3 = pam.build_mesh(3, (60, 220, 85), ((0, 1200), (0, 2200), (0, 170)))
    part3 = pam.make_partition(mesh3, 6, 22, 17)
    assert part3.n_subdomains == 2244
    np.testing.assert_array_equal(np.bincount(part3.cell_to_subdomain), [500] * 2244)
    assert part3.is_cell_aligned()
    with pytest.raises(ValueError):
        pam.build_mesh(4, (2, 2, 2, 2), ((0, 1),) * 4)


def test_boxes_cover_domain_once():
    mesh = pam.build_mesh(2, (16, 16), ((0, 1), (0, 1)))
    part = pam.make_partition(mesh, 4, 2)
    pts = np.random.default_rng(3).random((20000, 2))
    hits = sum(b.contains_many(pts).astype(int) for b in part.boxes)
    assert np.all(hits == 1)


def test_grid_edges_detection():
    mesh = pam.build_mesh(2, (8, 8), ((0, 1), (0, 1)))
    part = pam.make_partition(mesh, 2, 4)
    shape, edges = part.grid
    assert shape == (2, 4)
    np.testing.assert_array_equal(edges[1], np.arange(5) / 4)
    bad = (pam.Box(lo=(0.0,), hi=(0.6,), open_hi=(True,)), pam.Box(lo=(0.5,), hi=(1.0,), open_hi=(False,)))
    assert pam.geometry.grid_edges(bad) is None


def test_box_arrays_and_claimed_error_message():
    """Host side of the arbitrary-box path (geometry.py:54-66, 242-258): the box set as the
    C-ABI's (lo, hi, open_hi) arrays, and the reference's message for a doubly claimed point
    rebuilt from the device's packed (second box << 40 | point) key."""
    from paper_2605_16564_b200 import geometry as G

    boxes = (pam.Box(lo=(0.0, 0.0), hi=(0.5, 1.0), open_hi=(True, False)),
             pam.Box(lo=(0.5, 0.0), hi=(1.0, 1.0), open_hi=(False, False)),
             pam.Box(lo=(0.4, 0.4), hi=(0.6, 0.6), open_hi=(True, True)))
    assert G.grid_edges(boxes) is None
    lo, hi, op = G.box_arrays(boxes)
    assert lo.dtype == hi.dtype == np.float64 and op.dtype == np.int32
    assert lo.flags.c_contiguous and lo.shape == hi.shape == op.shape == (3, 2)
    np.testing.assert_array_equal(op, [[1, 0], [0, 0], [1, 1]])
    np.testing.assert_array_equal(hi[2], [0.6, 0.6])
    pts = np.array([[0.9, 0.9], [0.55, 0.55], [0.45, 0.45]])
    with pytest.raises(ValueError, match="^point index 1 claimed by boxes 1 and 2$"):
        G.raise_claimed((2 << 40) | 1, pts, boxes)
    with pytest.raises(ValueError, match="^point index 2 claimed by boxes 0 and 2$"):
        G.raise_claimed((2 << 40) | 2, pts, boxes)


def test_dictionary_capacity_matches_reference_loop_bounds():
    # C4: 500 + min(2*300, 599+300) = 1100; m_max=0 -> no growth
    cap = engine.dictionary_capacity([500, 500], [100, 100], [3, 3], [600, 0], [3, 3])
    np.testing.assert_array_equal(cap, [1100, 500])
    # box field criterion 5 (k_top=204, m_max=1836, 4 rounds): 1024 + 3*612 = 2860
    assert engine.dictionary_capacity([1024], [204], [3], [1836], [4])[0] == 2860
    # budget-limited: m_max=7, k*m_q=6 per round, 10 rounds: at most 6 + 6 = 12 added
    assert engine.dictionary_capacity([10], [2], [3], [7], [10])[0] == 22


def test_chunk_ranges():
    assert engine.chunk_ranges(np.array([5, 5, 5]), 100) == [(0, 3)]
    assert engine.chunk_ranges(np.array([5, 5, 5]), 10) == [(0, 2), (2, 3)]
    assert engine.chunk_ranges(np.array([50, 5]), 10) == [(0, 1), (1, 2)]


def test_lazy_checksum_metadata():
    field = pam.box_field_2d(4, 4)
    meta = _LazyChecksumMeta({"config": "x"}, field)
    assert "field_checksum" in meta
    assert meta["field_checksum"] == field.checksum()
    assert sorted(meta) == ["config", "field_checksum"]
    meta2 = _LazyChecksumMeta({"field_checksum": "given"}, None)
    assert meta2["field_checksum"] == "given"
    assert "field_checksum" not in _LazyChecksumMeta({}, None)


def _host_surrogate():
    field = pam.box_field_2d(8, 8)
    part = pam.make_partition(field.mesh, 2, 2)
    rng = np.random.default_rng(0)
    locs = []
    for b in part.boxes:
        c = np.asarray(b.lo) + rng.random((5, 2)) * 0.5
        d = pam.RbfDictionary(centers=c, widths=rng.uniform(0.05, 0.2, 5),
                              generations=np.array([0, 0, 0, 1, 2]))
        locs.append(pam.LocalSurrogate(dictionary=d, beta=rng.standard_normal(5)))
    return pam.GlobalSurrogate(partition=part, locals=tuple(locs), metadata={"config": "unit test"})


def test_save_load_roundtrip_text_identical(tmp_path):
    sur = _host_surrogate()
    text = pam.dumps(sur)
    back = pam.loads(text)
    assert pam.dumps(back) == text
    for a, b in zip(sur.locals, back.locals):
        np.testing.assert_array_equal(a.beta, b.beta)
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        np.testing.assert_array_equal(a.dictionary.generations, b.dictionary.generations)
    p = tmp_path / "s.txt"
    pam.save(sur, p)
    assert pam.dumps(pam.load(p)) == text


def test_load_errors():
    text = pam.dumps(_host_surrogate())
    with pytest.raises(pam.DataError, match="truncated"):
        pam.loads("\n".join(text.splitlines()[: len(text.splitlines()) // 2]))
    with pytest.raises(pam.DataError, match="not a surrogate"):
        pam.loads("something else entirely\n")
    with pytest.raises(pam.DataError, match="version"):
        pam.loads(text.replace("fieldfit-surrogate 1", "fieldfit-surrogate 99", 1))
    # one entry row short, the next one long by the same amount: the block total
    # still matches, the per-row check must catch it (reference partition.py:312)
    lines = text.splitlines()
    sub = next(k for k, ln in enumerate(lines) if ln.startswith("subdomain 0 "))
    a, b = lines[sub + 1].split(), lines[sub + 2].split()
    lines[sub + 1] = " ".join(a[:-1])
    lines[sub + 2] = " ".join(b + [a[-1]])
    with pytest.raises(pam.DataError, match="malformed dictionary entry at subdomain 0 row 0"):
        pam.loads("\n".join(lines) + "\n")


def test_reports_csv():
    reps = [pam.RoundReport(0, 16, 0, 0.5, 0.1, 0.2, 1.5, 0.01), pam.RoundReport(1, 22, 6, 0.25, 0.05, 0.1, 1.0, 0.02)]
    buf = io.StringIO()
    pam.reports_to_csv(reps, buf, provenance="cfg")
    lines = buf.getvalue().splitlines()
    assert lines[0] == "# cfg" and lines[1] == "round,centers,max_RT,rel_L2,objective,seconds"
    assert len(lines) == 4


def test_field_validation_and_checksum():
    mesh = pam.build_mesh(2, (2, 2), ((0, 1), (0, 1)))
    with pytest.raises(ValueError, match="cell 2"):
        pam.FieldData(mesh=mesh, values=np.array([1.0, 2.0, 0.0, 1.0]))
    f = pam.FieldData(mesh=mesh, values=np.array([1.0, 2.0, 3.0, 4.0]))
    assert f.checksum() == f.checksum()
    assert len(f.checksum()) == 64


def test_workload_shapes():
    from paper_2605_16564_b200 import workloads

    wl = workloads.config1()
    assert wl.field.mesh.n_cells == 4096 and wl.eval_points.shape == (16384, 2)
    p = workloads.config5(M=128, n_sub=8, n_eval=10)
    assert p.points.shape == (8000, 3) and p.centres.shape == (8 * 128, 3)
    assert np.all(p.points >= np.repeat(p.box_lo, 1000, axis=0))
    assert np.all(p.points < np.repeat(p.box_hi, 1000, axis=0))
    assert np.all(p.values > 0)


def test_save_byte_identical_to_reference_writer(golden):
    """dumps() reproduces the reference's text (partition.py:224-247) byte for byte."""
    from pathlib import Path

    g = golden("persistence")
    part = pam.make_partition(pam.build_mesh(2, (8, 6), ((0.0, 1.0), (-2.0, 1.0))), 2, 3)
    locs = tuple(
        pam.LocalSurrogate(dictionary=pam.RbfDictionary(centers=g[f"c{i}"], widths=g[f"w{i}"],
                                                        generations=g[f"g{i}"]), beta=g[f"b{i}"])
        for i in range(6))
    sur = pam.GlobalSurrogate(partition=part, locals=locs,
                              metadata={"config": "golden persistence", "field_checksum": "abc"})
    ref = (Path(__file__).parent / "golden" / "surrogate_ref.txt").read_text()
    assert pam.dumps(sur) == ref
    back = pam.loads(ref)
    assert pam.dumps(back) == ref
    for a, b in zip(back.locals, locs):
        np.testing.assert_array_equal(a.beta, b.beta)
