"""The drop-in claim, compiled: a C++20 caller written against the
reference's streamtune names (and the solver C ABI) builds against include/
and links libpm_tridiag.so; it runs its CPU part here, the solve on a GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _build(tmp_path):
    exe = tmp_path / "cpp_caller"
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
    cmd = [cxx, "-std=c++20", "-Wall", "-Wextra", "-Werror", str(ROOT / "examples" / "cpp_caller.cpp"),
           f"-I{ROOT / 'include'}", f"-L{ROOT / 'paper_2501_05938_b200'}", "-lpm_tridiag",
           f"-Wl,-rpath,{ROOT / 'paper_2501_05938_b200'}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_caller_builds_and_runs(tmp_path):
    out = subprocess.run([str(_build(tmp_path))], check=True, capture_output=True, text=True).stdout
    assert "benefit(8) 1.415968" in out  # PAPER.md:156 (Table 2)
    assert "caught InvalidStreamCountError(3)" in out
    assert "Eq. 2 bound holds: yes" in out
    assert "bundle round trip exact: yes; Table 4: 24 PASS, 0 FAIL, 1 KNOWN" in out


def test_c_header_is_plain_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "pm_tridiag.h"\n#include "streamtune_c.h"\nint main(void){return pm_get_version() > 0 ? 0 : 1;}\n')
    cc = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else "gcc"
    exe = tmp_path / "t"
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", str(src), f"-I{ROOT / 'include'}",
                    f"-L{ROOT / 'paper_2501_05938_b200'}", "-lpm_tridiag",
                    f"-Wl,-rpath,{ROOT / 'paper_2501_05938_b200'}", "-o", str(exe)], check=True)
    subprocess.run([str(exe)], check=True)


@pytest.mark.gpu
def test_cpp_caller_solves_on_gpu(tmp_path):
    out = subprocess.run([str(_build(tmp_path)), "--solve"], check=True, capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if l.startswith("solved")][0]
    assert float(line.split("residual")[1]) < 1e-12
    line = [l for l in out.splitlines() if l.startswith("fp32 status")][0].split()
    assert line[2] == "0" and float(line[5].rstrip(";")) < 1e-5
    assert line[8] == "0" and float(line[11]) < 1e-12
