"""Field ingestion (paper_2605_16564_b200.io) against the reference's io.py grammar."""

import io

import numpy as np
import pytest

import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import io as pio


def test_field_roundtrip_and_errors(tmp_path):
    field = pam.box_field_2d(6, 4)
    buf = io.StringIO()
    pio.write_field(field, buf)
    back = pio.read_field(io.StringIO(buf.getvalue()))
    np.testing.assert_array_equal(back.values, field.values)
    np.testing.assert_array_equal(back.mesh.centroids, field.mesh.centroids)
    p = tmp_path / "f.txt"
    pio.write_field(field, p)
    assert pio.read_field(p).mesh.counts == field.mesh.counts
    with pytest.raises(pam.DataError, match="too short"):
        pio.read_field(io.StringIO("2"))
    with pytest.raises(pam.DataError, match="header implies 4"):
        pio.read_field(io.StringIO("2 2 2\n0 1 0 1\n1 2 3\n"))
    with pytest.raises(pam.DataError, match="cell 2 is not positive"):
        pio.read_field(io.StringIO("1 3\n0 1\n1 2 -3\n"))
    with pytest.raises(pam.DataError, match="non-numeric value 'x' at cell 1"):
        pio.read_field(io.StringIO("1 3\n0 1\n1 x 3\n"))
    with pytest.raises(pam.DataError, match="cannot read"):
        pio.read_field(tmp_path / "missing.txt")


def _spe10_text(nz_used=85):
    rng = np.random.default_rng(0)
    vals = 10.0 ** rng.uniform(-3, 3, pio.SPE10_TOTAL_VALUES)
    return vals, " ".join(f"{v:.6e}" for v in vals)


def test_spe10_layer_and_3d():
    vals, text = _spe10_text()
    lay = pio.read_spe10(io.StringIO(text), 7)
    assert lay.mesh.counts == (60, 220)
    np.testing.assert_allclose(lay.values, vals[7 * 13200:8 * 13200], rtol=1e-6)
    f3 = pio.read_spe10_3d(io.StringIO(text), range(10, 14))
    assert f3.mesh.counts == (60, 220, 4) and f3.mesh.cell_size == (20.0, 10.0, 2.0)
    np.testing.assert_allclose(f3.values, vals[10 * 13200:14 * 13200], rtol=1e-6)
    assert f3.mesh.centroids[0, 2] == 20.0 + 1.0  # layer 10 -> z in [20, 22)
    with pytest.raises(pam.DataError, match="layer must lie"):
        pio.read_spe10(io.StringIO(text), 85)
    with pytest.raises(pam.DataError, match="exactly"):
        pio.read_spe10(io.StringIO("1 2 3"), 0)
    bad = text.split()
    bad[5 * 13200 + 3] = "-1"
    with pytest.raises(pam.DataError, match=f"offset {5 * 13200 + 3} is not positive"):
        pio.read_spe10(io.StringIO(" ".join(bad)), 5)


def test_write_grid_csv_matches_reference_layout():
    buf = io.StringIO()
    pam.write_grid_csv(np.array([[0.5, 0.25], [1.0, 2.0]]), [1.5, 2.5], buf, provenance="cfg")
    assert buf.getvalue() == "# cfg\nx,y,value\n0.5,0.25,1.5\n1,2,2.5\n"
    buf = io.StringIO()
    pam.write_grid_csv(np.zeros((1, 3)), [3.0], buf)
    assert buf.getvalue() == "x,y,z,value\n0,0,0,3\n"
    with pytest.raises(ValueError, match="2 points but 1 values"):
        pam.write_grid_csv(np.zeros((2, 2)), [1.0], io.StringIO())
