"""`python -m paper_2007_06048_b200 model ...` -- the reference's `minimod model`
front end (ref: tools/cli.cpp:60-101, 256-272) on the B200 engine.

Same flags and output for the acoustic_iso_cd path (and acoustic_iso, the
variable-density engine): the parameter block, the run, the timing lines, and
the shot record (raw f32 + JSON sidecar) when --output is given.  Exit codes as the reference: 2 for configuration errors,
3 for anything else.  `--kernels fast|strict` selects the kernel family (both
bit-identical to the CPU reference); `--device` the GPU.
"""
from __future__ import annotations

import argparse
import sys

from ._lib import ConfigError


def _tuple(flag: str, value: str, kind, n: int = 3):
    cells = value.split(",")
    if len(cells) != n:
        raise ConfigError(f"{flag} expects {n} comma-separated values, got '{value}'")
    try:
        return tuple(kind(c) for c in cells)
    except ValueError:
        raise ConfigError(f"{flag}: cannot parse '{value}'") from None


def parse(argv):
    if not argv or argv[0].startswith("-"):
        raise ConfigError("missing subcommand (valid: model)")
    sub, rest = argv[0], argv[1:]
    if sub != "model":
        raise ConfigError(f"unknown subcommand '{sub}' (valid: model; multi-GPU runs go "
                          "through paper_2007_06048_b200.dist under torchrun)")
    ap = argparse.ArgumentParser(prog="python -m paper_2007_06048_b200 model", add_help=False)
    ap.add_argument("--ngrid", default="100,100,100")
    ap.add_argument("--dgrid", default="20,20,20")
    ap.add_argument("--nsteps", type=int, default=1000)
    ap.add_argument("--fmax", type=float, default=25.0)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--propagator", default="acoustic_iso_cd")
    ap.add_argument("--free-surface", action="store_true")
    ap.add_argument("--model-manifest", default="")
    ap.add_argument("--output", default="")
    ap.add_argument("--kernels", default="fast", choices=["fast", "strict"])
    ap.add_argument("--device", type=int, default=0)
    try:
        a, unknown = ap.parse_known_args(rest)
    except SystemExit:
        raise ConfigError("cannot parse the command line") from None
    if unknown:
        raise ConfigError(f"unknown arguments: {' '.join(unknown)}")
    if a.propagator not in ("acoustic_iso_cd", "acoustic_iso"):
        raise ConfigError(f"--propagator {a.propagator}: this build serves acoustic_iso_cd and "
                          "acoustic_iso")
    a.ngrid = _tuple("--ngrid", a.ngrid, int)
    a.dgrid = _tuple("--dgrid", a.dgrid, float)
    if a.nsteps < 1:
        raise ConfigError("--nsteps must be >= 1")
    if a.fmax <= 0.0:
        raise ConfigError("--fmax must be > 0")
    if any(n < 1 for n in a.ngrid):
        raise ConfigError("--ngrid entries must be >= 1")
    if any(not d > 0.0 for d in a.dgrid):
        raise ConfigError("--dgrid entries must be > 0")
    return a


def main(argv=None, out=sys.stdout, err=sys.stderr) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if argv and argv[0] in ("-h", "--help", "help"):
        out.write(__doc__)
        return 0
    try:
        a = parse(argv)
    except ConfigError as e:
        err.write(f"error: {e}\n")
        return 2
    try:
        from . import driver, numerics, shotio
        cfg = driver.SimConfig(propagator=a.propagator, ngrid=a.ngrid, dgrid=a.dgrid,
                               nsteps=a.nsteps, fmax=a.fmax, free_surface=a.free_surface)
        grid = numerics.make_grid(cfg.ngrid, cfg.dgrid, cfg.stencil_radius)
        if a.model_manifest:
            model = shotio.load_model(a.model_manifest, cfg.stencil_radius)
            if tuple(model.grid.n) != tuple(cfg.ngrid):
                raise ConfigError("model manifest grid does not match --ngrid")
        else:
            model = numerics.default_layered_model(grid)
        out.write(driver.render_parameter_block(cfg, model))
        rec, rep = driver.run(cfg, model, device=a.device, mode=a.kernels)
        out.write(driver.render_timing(rep))
        if a.output:
            shotio.save_record(rec, a.output)
        return 0
    except ConfigError as e:
        err.write(f"error: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 -- the reference maps the rest to 3
        err.write(f"error: {e}\n")
        return 3


if __name__ == "__main__":
    sys.exit(main())
