"""File formats around the solve: PGM/PPM/PNG in, .flo/PFM out, key=value
EnergyParams, calibration. Host-side only; SPEC.md's invariants as tests."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200 import fileio
from paper_1610_07159_b200.hwflow import EnergyParams, FlowResult


def test_flo_round_trip_is_bit_identical(tmp_path):
    """SPEC.md:537 `.flo files written ... read back bit-identically`."""
    rng = np.random.default_rng(0)
    uv = rng.normal(0, 3, (17, 23, 2)).astype(np.float32)
    fileio.write_flo(tmp_path / "a.flo", uv)
    raw = (tmp_path / "a.flo").read_bytes()
    assert raw[:4] == b"PIEH" and len(raw) == 12 + 17 * 23 * 8
    assert np.array_equal(fileio.read_flo(tmp_path / "a.flo"), uv)


def test_pfm_round_trip(tmp_path):
    a = np.arange(12, dtype=np.float32).reshape(3, 4) - 5.5
    fileio.write_pfm(tmp_path / "d.pfm", a)
    assert (tmp_path / "d.pfm").read_bytes().startswith(b"Pf\n4 3\n-1.0\n")
    assert np.array_equal(fileio.read_pfm(tmp_path / "d.pfm"), a)


def test_pgm_ppm_png_normalisation(tmp_path):
    """normalised by the format max; color -> luma 0.299/0.587/0.114."""
    g8 = np.arange(30, dtype=np.uint8).reshape(5, 6) * 8
    fileio.write_pgm(tmp_path / "g8.pgm", g8)
    r = fileio.read_image(tmp_path / "g8.pgm")
    assert r.dtype == np.uint8 and np.array_equal(r, g8)  # exact k/255 on the device
    g16 = (np.arange(30, dtype=np.uint16).reshape(5, 6) * 2000)
    fileio.write_pgm(tmp_path / "g16.pgm", g16)
    assert np.array_equal(fileio.read_image(tmp_path / "g16.pgm"), g16 / 65535.0)
    rgb = np.zeros((2, 3, 3), np.uint8)
    rgb[..., 0], rgb[..., 1], rgb[..., 2] = 255, 0, 255
    (tmp_path / "c.ppm").write_bytes(b"P6\n# comment\n3 2\n255\n" + rgb.tobytes())
    assert np.allclose(fileio.read_image(tmp_path / "c.ppm"), 0.299 + 0.114)
    from PIL import Image
    Image.fromarray(g8).save(tmp_path / "g8.png")
    assert np.array_equal(fileio.read_image(tmp_path / "g8.png"), g8)


def test_params_round_trip_and_errors():
    """parse(serialize(config)) = config; unknown keys rejected."""
    for name in ("live", "facial", "stereo-hq"):
        p = EnergyParams.preset(name)
        assert fileio.parse_params(fileio.dump_params(p)) == p
    p = fileio.parse_params("preset = facial\nw_epi=0.25  # comment\n")
    assert p.w_epi == 0.25 and p.w_grad == 5.0
    with pytest.raises(ValueError, match="unknown key"):
        fileio.parse_params("w_nope=1\n")
    with pytest.raises(ValueError, match=">= 0"):
        fileio.parse_params("w_reg=-1\n")


def test_write_flow_result(tmp_path):
    r = FlowResult(4, 3)
    r.s = np.ones((3, 4, 2))
    r.m = np.zeros((3, 4, 2))
    r.d = np.full((3, 4, 2), -0.5)
    r.disparity = 2.0 * r.s[..., 0]
    paths = fileio.write_flow_result(tmp_path, r, "f0")
    assert [p.name for p in paths] == ["f0_s.flo", "f0_m.flo", "f0_d.flo", "f0_disparity.pfm"]
    assert np.array_equal(fileio.read_flo(paths[2]), r.d.astype(np.float32))
    assert np.array_equal(fileio.read_pfm(paths[3]), np.full((3, 4), 2.0, np.float32))
