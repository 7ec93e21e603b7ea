"""Shot records and velocity models in the reference's on-disk formats.

SURVEY.md §8(f) rows 1 and 3:

* shot record -- ``save_record`` (ref: source.cpp:68-95): raw little-endian
  f32 traces ``[nreceivers x nsteps]`` (trace r, sample s at r*nsteps+s) plus a
  JSON sidecar ``<path>.json`` {dt, nsteps, nreceivers, source_loc,
  receiver_increment, nshots}; both written to ``.tmp`` files and renamed, so
  a reader never sees a partial file.
* model -- ``load_model`` / ``save_model`` (ref: model.cpp:64-190): a JSON
  manifest {n, d, components{vp: file}, dtype "f32le", order "z-fastest"}
  next to headerless f32 volumes of the interior, z fastest; loading validates
  the model and replicates the ghosts (validate_model, model.cpp:15-43).

Host code only (numpy); the layouts are pinned against the reference's own
writers in tests/test_shotio.py.
"""
from __future__ import annotations

import json
import math
import os
from pathlib import Path

import numpy as np

from ._lib import ConfigError
from .numerics import AcquisitionGeometry, EarthModel, ShotRecord, make_grid, validate_model


# ------------------------------------------------------------------ JSON
def _num(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    v = float(v)
    if not math.isfinite(v):
        raise ConfigError("non-finite number in a JSON file")
    return repr(v)  # shortest round-trip decimal, like nlohmann's dtoa


def _dump(v, ind: int = 0) -> str:
    """JSON in the layout of nlohmann's ``dump(2)`` as the reference writes it:
    sorted keys, two-space indent, integer arrays inline, other arrays one
    element per line."""
    pad = " " * ind
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad}  {json.dumps(str(k))}: {_dump(v[k], ind + 2)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        if all(isinstance(x, (int, np.integer)) and not isinstance(x, bool) for x in v):
            return "[" + ",".join(str(int(x)) for x in v) + "]"
        return "[\n" + ",\n".join(f"{pad}  {_dump(x, ind + 2)}" for x in v) + "\n" + pad + "]"
    if isinstance(v, str):
        return json.dumps(v)
    return _num(v)


def _write_atomic(path: Path, data: bytes) -> Path:
    tmp = Path(str(path) + ".tmp")
    try:
        with open(tmp, "wb") as f:
            f.write(data)
    except OSError as e:
        raise ConfigError(f"cannot write {path}: {e}") from e
    return tmp


# ------------------------------------------------------------------ shot records
def save_record(record: ShotRecord, path) -> None:
    """ref: source.cpp:68-95 -- traces, then the sidecar; both renamed last."""
    path = str(path)
    if not path:
        raise ConfigError("empty output path")
    traces = np.ascontiguousarray(record.traces, dtype="<f4")
    g = record.geometry
    if traces.shape != (g.nreceivers(), record.nsteps):
        raise ConfigError("trace matrix must be [nreceivers x nsteps]")
    side = {
        "dt": float(record.dt),
        "nsteps": int(record.nsteps),
        "nreceivers": int(g.nreceivers()),
        "source_loc": [int(x) for x in g.source_loc],
        "receiver_increment": [int(x) for x in g.receiver_increment],
        "nshots": int(g.nshots),
    }
    data_tmp = _write_atomic(Path(path), traces.tobytes())
    side_tmp = _write_atomic(Path(path + ".json"), (_dump(side) + "\n").encode())
    os.replace(data_tmp, path)
    os.replace(side_tmp, path + ".json")


def load_record(path) -> ShotRecord:
    """Inverse of save_record (receiver coordinates are not part of the format)."""
    path = str(path)
    try:
        side = json.loads(Path(path + ".json").read_text())
        raw = np.fromfile(path, dtype="<f4")
    except (OSError, ValueError) as e:
        raise ConfigError(f"cannot read shot record {path}: {e}") from e
    nrec, nsteps = int(side["nreceivers"]), int(side["nsteps"])
    if raw.size != nrec * nsteps:
        raise ConfigError(f"size mismatch for {path}: sidecar implies {nrec * nsteps * 4} "
                          f"bytes, file has {raw.size * 4}")
    geo = AcquisitionGeometry(tuple(side["source_loc"]),
                              np.zeros((nrec, 3), np.int32),
                              tuple(side["receiver_increment"]), nshots=int(side["nshots"]))
    return ShotRecord(nsteps, float(side["dt"]), geo,
                      raw.astype(np.float32).reshape(nrec, nsteps))


# ------------------------------------------------------------------ models
def save_model(model: EarthModel, manifest) -> None:
    """ref: model.cpp:157-184 (vp, and rho when the model has one)."""
    manifest = Path(manifest)
    if not str(manifest):
        raise ConfigError("empty model manifest path")
    g = model.grid
    comps = {}
    for name, field in (("vp", model.vp), ("rho", model.rho)):
        if field is None:
            continue
        vol = np.ascontiguousarray(g.inner(np.asarray(field, dtype=np.float32)), dtype="<f4")
        path = manifest.parent / f"{name}.f32"
        os.replace(_write_atomic(path, vol.tobytes()), path)
        comps[name] = f"{name}.f32"
    man = {"n": [int(x) for x in g.n], "d": [float(x) for x in g.d],
           "components": comps, "dtype": "f32le", "order": "z-fastest"}
    os.replace(_write_atomic(manifest, (_dump(man) + "\n").encode()), manifest)


def _read_volume(path: Path, grid, count: int) -> np.ndarray:
    try:
        nbytes = path.stat().st_size
    except OSError as e:
        raise ConfigError(f"cannot open volume file: {path}") from e
    if nbytes != 4 * count:
        raise ConfigError(f"size mismatch for {path}: manifest implies {4 * count} bytes, "
                          f"file has {nbytes}")
    f = grid.field()
    grid.inner(f)[...] = np.fromfile(path, dtype="<f4").reshape(grid.n)
    return f


def load_model(manifest, radius: int = 4) -> EarthModel:
    """ref: model.cpp:122-155 -- manifest + f32 volumes -> validated, ghosted
    vp (and rho when the manifest lists one; vs is elastic-only and ignored)."""
    manifest = Path(manifest)
    if not str(manifest):
        raise ConfigError("empty model manifest path")
    try:
        j = json.loads(manifest.read_text())
    except OSError as e:
        raise ConfigError(f"cannot open model manifest: {manifest}") from e
    except ValueError as e:
        raise ConfigError(f"malformed model manifest {manifest}: {e}") from e
    if j.get("dtype", "f32le") != "f32le":
        raise ConfigError("unsupported dtype in manifest (only f32le)")
    if j.get("order", "z-fastest") != "z-fastest":
        raise ConfigError("unsupported order in manifest (only z-fastest)")
    try:
        n = tuple(int(x) for x in j["n"])
        d = tuple(float(x) for x in j["d"])
        comps = j["components"]
        vp_file = manifest.parent / comps["vp"]
        rho_file = manifest.parent / comps["rho"] if "rho" in comps else None
    except (KeyError, TypeError) as e:
        raise ConfigError(f"malformed model manifest {manifest}: missing {e}") from e
    grid = make_grid(n, d, radius)
    count = n[0] * n[1] * n[2]
    vp = _read_volume(vp_file, grid, count)
    rho = _read_volume(rho_file, grid, count) if rho_file is not None else None
    return validate_model(EarthModel(grid, vp, rho=rho))
