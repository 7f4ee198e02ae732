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


def _build_dist(tmp_path):
    exe = tmp_path / "dist_caller"
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
    cuda = Path("/usr/local/cuda")
    cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", str(ROOT / "examples" / "dist_caller.cpp"),
           f"-I{ROOT / 'include'}", f"-I{cuda / 'include'}", f"-L{ROOT / 'paper_2501_05938_b200'}",
           f"-L{cuda / 'lib64'}", "-lpm_tridiag", "-lcudart", "-lpthread",
           f"-Wl,-rpath,{ROOT / 'paper_2501_05938_b200'}", f"-Wl,-rpath,{cuda / 'lib64'}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    return exe


def test_dist_caller_builds(tmp_path):
    """The C++ row-sharded caller (pm_solve_dist_* with a caller-supplied
    all-gather, pm_nccl_*) compiles against include/ and links."""
    assert _build_dist(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n", [(1, 1000), (2, 1_000_003), (3, 777_777), (8, 5_000_001)])
def test_dist_caller_host_staged_allgather(tmp_path, world, n):
    """`world` ranks as threads on one GPU through pm_solve_dist_f64 with a
    host-staged all-gather callback: x matches the single-system solve and
    meets the residual bar."""
    out = subprocess.run([str(_build_dist(tmp_path)), str(world), str(n)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("dist world")][0].split()
    assert float(line[6]) <= 1e-10 and float(line[8]) <= 1e-12, line
    assert out.stdout.count("status 0") == world


@pytest.mark.gpu
def test_dist_caller_nccl_one_rank(tmp_path):
    """pm_solve_dist_nccl_f64 on a one-rank communicator made by pm_nccl_*
    (NCCL dlopen'ed by the library): the ncclAllGather path end to end."""
    out = subprocess.run([str(_build_dist(tmp_path)), "--nccl", "2000003"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert int(out.stdout.split("nccl version")[1].split()[0]) >= 21800
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("dist world")][0].split()
    assert float(line[6]) <= 1e-10 and float(line[8]) <= 1e-12, line
