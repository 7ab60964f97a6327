"""Verification tooling (NEXT-4): Eq. 6 matching digits and MPXD dump
comparison, the methodology of PAPER.md §3.1 (Fig. 5).

  digits(ref, other)      Eq. 6: -log10(|ref - other| / |ref|), 16 for
                          an exact match, clamped to [-5, 16]; NaN where
                          ref == 0 (Fig. 5 compares non-zero quantities).
  histogram(d)            integer-binned counts of a digits array (bins -5..16).
  read_dump(path)         MPXD file (written by mfx_state_dump, layout in
                          include/mfx.h / DESIGN.md §13) -> header + arrays.
  compare_dumps(a, b)     per-field digits histograms and min / median / mode.

Host-side numpy analysis of files: nothing here is on the GPU hot path.
"""
from __future__ import annotations

import struct

import numpy as np

HEADER = struct.Struct("<4sIiiiqddI")     # magic, version, nx, ny, nz, n_parcels, time, dt, n_fields
ENTRY = struct.Struct("<8sB7x")           # name, kind (0 cell, 1 parcel)
BINS = np.arange(-5, 17)


def digits(ref, other):
    """Eq. 6 element-wise."""
    ref = np.asarray(ref, dtype=np.float64)
    other = np.asarray(other, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        d = -np.log10(np.abs(ref - other) / np.abs(ref))
    d = np.where(ref == other, 16.0, d)
    d = np.clip(d, -5.0, 16.0)
    return np.where(ref == 0.0, np.nan, d)


def histogram(d):
    """Counts per integer bin -5..16 (digits rounded to the nearest integer, as
    Fig. 5's bars); NaNs (zero references) are excluded and counted separately."""
    d = np.asarray(d, dtype=np.float64)
    ok = ~np.isnan(d)
    b = np.clip(np.rint(d[ok]).astype(np.int64), -5, 16)
    counts = np.bincount(b + 5, minlength=len(BINS))
    return {int(k): int(c) for k, c in zip(BINS, counts)}, int((~ok).sum())


def read_dump(path: str) -> dict:
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, ver, nx, ny, nz, npar, t, dt, nf = HEADER.unpack_from(raw, 0)
    if magic != b"MPXD":
        raise ValueError(f"{path}: bad magic")
    if ver != 1:
        raise ValueError(f"{path}: unsupported version {ver}")
    off = HEADER.size
    table = []
    for _ in range(nf):
        if off + ENTRY.size > len(raw):
            raise ValueError(f"{path}: truncated field table")
        name, kind = ENTRY.unpack_from(raw, off)
        table.append((name.rstrip(b"\0").decode(), kind))
        off += ENTRY.size
    n = nx * ny * nz
    fields = {}
    for name, kind in table:
        cnt = npar if kind else n
        if off + 8 * cnt > len(raw):
            raise ValueError(f"{path}: truncated payload ({name})")
        fields[name] = np.frombuffer(raw, dtype="<f8", count=cnt, offset=off).copy()
        off += 8 * cnt
    return dict(dims=(nx, ny, nz), n_parcels=npar, time=t, dt=dt, fields=fields)


def write_dump(path: str, dims, fields: dict, parcels: dict | None = None, time: float = 0.0, dt: float = 0.0):
    """Writer of the same layout (host arrays), for tools and tests."""
    nx, ny, nz = dims
    npar = len(next(iter(parcels.values()))) if parcels else 0
    items = [(k, 0, np.asarray(v, dtype="<f8")) for k, v in fields.items()]
    items += [(k, 1, np.asarray(v, dtype="<f8")) for k, v in (parcels or {}).items()]
    with open(path, "wb") as f:
        f.write(HEADER.pack(b"MPXD", 1, nx, ny, nz, npar, time, dt, len(items)))
        for k, kind, _ in items:
            f.write(ENTRY.pack(k.encode()[:8], kind))
        for _, _, a in items:
            f.write(np.ascontiguousarray(a).tobytes())


def compare_dumps(path_ref: str, path_other: str) -> dict:
    """per-field Eq. 6 histograms of two dumps of the same grid."""
    a, b = read_dump(path_ref), read_dump(path_other)
    if a["dims"] != b["dims"] or a["n_parcels"] != b["n_parcels"]:
        raise ValueError("dumps differ in shape")
    out = {}
    for name, ra in a["fields"].items():
        if name not in b["fields"]:
            continue
        d = digits(ra, b["fields"][name])
        hist, zeros = histogram(d)
        ok = d[~np.isnan(d)]
        out[name] = {"hist": hist, "zero_refs": zeros,
                     "min": float(ok.min()) if ok.size else None,
                     "median": float(np.median(ok)) if ok.size else None,
                     "mode": max(hist, key=hist.get) if ok.size else None}
    return out
