"""The C-ABI library loads and exports every symbol include/minimod_b200.h
declares; error codes map to the reference's exception types.  CPU only."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "minimod_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(mm):
    from paper_2007_06048_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding knows every one of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_library_is_sm100a(mm):
    import subprocess
    from paper_2007_06048_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.loaded_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_cxx_header_compiles(tmp_path):
    """include/minimod_b200.hpp (the C++ drop-in wrapper) compiles standalone."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text('#include "minimod_b200.hpp"\nint main(){ minimod_b200::EngineOptions o; '
                   'minimod_b200::AcousticVdEngine* e = nullptr; (void)e; '
                   'return o.ndamping[0]; }\n')
    res = subprocess.run([gxx, "-std=c++17", "-fsyntax-only", f"-I{ROOT / 'include'}", str(src)],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_error_mapping_without_gpu(mm):
    import numpy as np
    g = mm.make_grid((12, 12, 12), (10, 10, 10))
    vp = g.field(1500.0)
    if mm.device_count() == 0:
        with pytest.raises(mm.CudaError, match="GPU"):
            mm.AcousticCdEngine(g, (0, 0, 0), g.n, vp)
    with pytest.raises(mm.ConfigError):
        mm.ricker(25.0, -1.0, 3)
    with pytest.raises(ValueError):
        from paper_2007_06048_b200 import _lib
        _lib.check(_lib.lib().mm_cd_step(None, 0.0, None))


def _env_after_import(env):
    code = (f"import os, sys; sys.path.insert(0, {str(ROOT)!r}); import paper_2007_06048_b200;"
            "print(os.environ['CUDA_DEVICE_MAX_CONNECTIONS'])")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=300)
    return out.stdout.strip(), out.stderr[-500:]


def test_package_raises_hardware_queue_default():
    """Importing the package asks for 32 CUDA hardware connections unless the
    user chose a value (several engines per process otherwise share queues and
    serialise their side streams)."""
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    got, err = _env_after_import(env)
    assert got == "32", err
    got, err = _env_after_import({**env, "CUDA_DEVICE_MAX_CONNECTIONS": "4"})
    assert got == "4", err
