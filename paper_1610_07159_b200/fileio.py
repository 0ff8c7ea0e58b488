"""File formats around the solve.

This is host-side I/O only; the CLI itself is out of scope.
  - Images: binary PGM/PPM (P5/P6, 8 or 16 bit), parsed here; PNG through PIL. Color is
    converted to luma 0.299/0.587/0.114, and intensities are normalised by the
    format's maximum. 8-bit gray stays uint8, so the device computes k/255
    exactly as the reference does; everything else becomes float64 in [0, 1].
  - Flow: Middlebury .flo (magic "PIEH" = 202021.25f, int32 width and height, then float32
    u, v interleaved, little-endian). s, m and d are written as three files.
  - Disparity/depth: PFM ("Pf", one channel, negative scale = little-endian, rows bottom-up).
  - EnergyParams: key=value text with Table 1 names; parse(serialize(p)) == p.
  - Calibration: StereoRig.load (hwflow.py), 9 or 9 + 24 numbers.
"""
from __future__ import annotations

import re
from dataclasses import fields
from pathlib import Path

import numpy as np

from .hwflow import EnergyParams, FlowResult

FLO_MAGIC = 202021.25
LUMA = (0.299, 0.587, 0.114)


def _luma(rgb: np.ndarray) -> np.ndarray:
    return rgb[..., 0] * LUMA[0] + rgb[..., 1] * LUMA[1] + rgb[..., 2] * LUMA[2]


def read_pnm(path: str | Path) -> np.ndarray:
    """Binary PGM (P5) / PPM (P6), maxval <= 65535 (big-endian 16 bit, per the Netpbm spec)."""
    data = Path(path).read_bytes()
    tokens, pos = [], 0
    while len(tokens) < 4:
        m = re.compile(rb"\s*(#[^\n]*\n\s*)*(\S+)").match(data, pos)
        if not m:
            raise ValueError(f"{path}: truncated PNM header")
        tokens.append(m.group(2))
        pos = m.end()
    magic, w, h, maxval = tokens[0], int(tokens[1]), int(tokens[2]), int(tokens[3])
    if magic not in (b"P5", b"P6") or not 0 < maxval < 65536:
        raise ValueError(f"{path}: not a binary PGM/PPM")
    pos += 1  # the single whitespace byte after maxval
    ch = 3 if magic == b"P6" else 1
    dt = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
    n = w * h * ch
    raw = np.frombuffer(data, dtype=dt, count=n, offset=pos)
    img = raw.reshape(h, w, ch) if ch == 3 else raw.reshape(h, w)
    if ch == 1 and maxval == 255:
        return img.copy()
    v = img.astype(np.float64) / maxval
    return _luma(v) if ch == 3 else v


def read_image(path: str | Path) -> np.ndarray:
    """(h, w) uint8 (8-bit gray) or float64 in [0, 1] (16-bit or color)."""
    p = Path(path)
    if p.suffix.lower() in (".pgm", ".ppm", ".pnm"):
        return read_pnm(p)
    from PIL import Image  # PNG and the rest
    with Image.open(p) as im:
        if im.mode == "L":
            return np.asarray(im, dtype=np.uint8).copy()
        if im.mode in ("I;16", "I;16B", "I;16L", "I"):
            a = np.asarray(im).astype(np.float64)
            return a / 65535.0
        if im.mode in ("RGB", "RGBA", "P", "LA"):
            a = np.asarray(im.convert("RGB"), dtype=np.float64) / 255.0
            return _luma(a)
        raise ValueError(f"{path}: unsupported image mode {im.mode}")


def write_pgm(path: str | Path, img: np.ndarray) -> None:
    """8-bit (uint8) or 16-bit (uint16) binary PGM."""
    a = np.asarray(img)
    if a.dtype == np.uint8:
        body, maxval = a.tobytes(), 255
    elif a.dtype == np.uint16:
        body, maxval = a.astype(">u2").tobytes(), 65535
    else:
        raise ValueError("write_pgm takes uint8 or uint16")
    Path(path).write_bytes(f"P5\n{a.shape[1]} {a.shape[0]}\n{maxval}\n".encode() + body)


def write_flo(path: str | Path, uv: np.ndarray) -> None:
    """Middlebury .flo of an (h, w, 2) flow."""
    a = np.asarray(uv)
    if a.ndim != 3 or a.shape[2] != 2:
        raise ValueError("flow must be (h, w, 2)")
    h, w = a.shape[:2]
    with open(path, "wb") as f:
        np.array([FLO_MAGIC], "<f4").tofile(f)
        np.array([w, h], "<i4").tofile(f)
        a.astype("<f4").tofile(f)


def read_flo(path: str | Path) -> np.ndarray:
    with open(path, "rb") as f:
        if np.fromfile(f, "<f4", 1)[0] != np.float32(FLO_MAGIC):
            raise ValueError(f"{path}: bad .flo magic")
        w, h = np.fromfile(f, "<i4", 2)
        return np.fromfile(f, "<f4", int(w) * int(h) * 2).reshape(int(h), int(w), 2)


def write_pfm(path: str | Path, img: np.ndarray) -> None:
    """One-channel little-endian PFM (rows stored bottom-up)."""
    a = np.asarray(img, np.float32)
    h, w = a.shape
    with open(path, "wb") as f:
        f.write(f"Pf\n{w} {h}\n-1.0\n".encode())
        a[::-1].astype("<f4").tofile(f)


def read_pfm(path: str | Path) -> np.ndarray:
    with open(path, "rb") as f:
        if f.readline().strip() != b"Pf":
            raise ValueError(f"{path}: not a one-channel PFM")
        w, h = (int(t) for t in f.readline().split())
        scale = float(f.readline())
        a = np.fromfile(f, "<f4" if scale < 0 else ">f4", w * h).reshape(h, w)
        return a[::-1].copy()


def write_flow_result(out_dir: str | Path, result: FlowResult, stem: str = "frame") -> list[Path]:
    """cli_flow outputs: s/m/d .flo files and the disparity PFM."""
    d = Path(out_dir)
    d.mkdir(parents=True, exist_ok=True)
    paths = []
    for name in ("s", "m", "d"):
        v = getattr(result, name)
        if v is not None:
            paths.append(d / f"{stem}_{name}.flo")
            write_flo(paths[-1], v)
    if result.disparity is not None:
        paths.append(d / f"{stem}_disparity.pfm")
        write_pfm(paths[-1], result.disparity)
    return paths


def dump_params(p: EnergyParams) -> str:
    """key=value lines, Table 1 names (energy.hpp:17-27), repr-exact doubles."""
    return "".join(f"{f.name}={getattr(p, f.name)!r}\n" for f in fields(p))


def parse_params(text: str, base: EnergyParams | None = None) -> EnergyParams:
    """Inverse of dump_params. Unknown keys are rejected; '#' starts a comment;
    'preset=name' starts from that preset."""
    known = {f.name for f in fields(EnergyParams)}
    kv = []
    for ln, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"line {ln}: expected key=value")
        k, v = (t.strip() for t in line.split("=", 1))
        kv.append((ln, k, v))
    p = base if base is not None else EnergyParams()
    for ln, k, v in kv:
        if k == "preset":
            p = EnergyParams.preset(v)
    vals = {f.name: getattr(p, f.name) for f in fields(EnergyParams)}
    for ln, k, v in kv:
        if k == "preset":
            continue
        if k not in known:
            raise ValueError(f"line {ln}: unknown key {k!r}")
        vals[k] = float(v)
    out = EnergyParams(**vals)
    out.validate()
    return out


def load_params(path: str | Path) -> EnergyParams:
    return parse_params(Path(path).read_text())
