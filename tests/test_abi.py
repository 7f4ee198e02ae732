"""CPU tests of the C-ABI boundary: the native library loads, exports every
symbol include/*.h declares, and the calls that need no GPU behave."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    names = set()
    for h in ("pm_tridiag.h", "streamtune_c.h"):
        text = (ROOT / "include" / h).read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s+((?:pm|st)_[a-z0-9_]+)\s*\(", text,
                             flags=re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_api():
    names = declared_functions()
    for must in ("pm_create", "pm_destroy", "pm_solve_host_f64", "pm_solve_device_f64",
                 "pm_solve_batch_device_f64", "pm_dist_reduce_f64", "pm_dist_solve_f64",
                 "pm_recommend_streams", "st_recommend", "st_fit_bundle", "st_overlap_sum"):
        assert must in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol():
    from paper_2501_05938_b200 import _lib

    L = _lib.load()
    missing = [n for n in sorted(declared_functions()) if not hasattr(L, n)]
    assert missing == []
    bound = {name for name, _, _ in _lib.PM_SIGNATURES}
    assert declared_functions() == bound


def test_library_is_built_for_sm100a():
    import subprocess

    lib = ROOT / "paper_2501_05938_b200" / "libpm_tridiag.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2501_05938_b200 import CudaRuntimeError, PartitionSolver

    with pytest.raises(CudaRuntimeError):
        PartitionSolver(0)


def test_pure_host_entry_points():
    from paper_2501_05938_b200 import _lib, recommend_streams

    L = _lib.load()
    assert L.pm_get_version() >= 100
    assert recommend_streams(10**6) == 8
    assert L.pm_recommend_streams(0, None) == -1
    b = _lib.ModelBundleC()
    assert L.pm_paper_bundle(C.byref(b)) == 0 and b.num_candidates == 5
    bad = _lib.ModelBundleC(*([0.0] * 8), 1000, 2)
    bad.candidates[0], bad.candidates[1] = 4, 2  # not increasing
    assert L.pm_recommend_streams(1000, C.byref(bad)) == -1


def test_python_package_does_not_import_oracle():
    pkg = ROOT / "paper_2501_05938_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
    for f in list((pkg / "csrc").rglob("*.c*")) + list((pkg / "csrc").rglob("*.h")):
        assert not re.search(r'#\s*include\s*[<"][^>"]*oracle', f.read_text()), f
    out = __import__("subprocess").run(["ldd", str(pkg / "libpm_tridiag.so")], capture_output=True,
                                       text=True).stdout
    assert "oracle" not in out
