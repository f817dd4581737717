"""Deadlock freedom of the batched tile-Cholesky ticket order (CPU).

tools/taskmap_check.cu links the built library and, for batches of
consecutive slot-ordered slimLS steps with tile reuse (configs[0..4] shapes
and edge shapes: blocks smaller than a tile, r = 0, r = 31, ell = 1, a
damping change mid-run), checks that every fresh tile has a task and every
dependency of every task is produced at a smaller ticket.
"""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1912_07962_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not (os.path.exists(NVCC) or shutil.which("nvcc")), reason="nvcc not available")
def test_ticket_order_respects_dependencies(tmp_path):
    lib = os.path.join(PKG, "libslimb200.so")
    if not os.path.exists(lib):
        pytest.skip("library not built")
    exe = tmp_path / "taskmap_check"
    nvcc = NVCC if os.path.exists(NVCC) else shutil.which("nvcc")
    subprocess.run([nvcc, "-std=c++17", "-arch=sm_100a", "-I", os.path.join(PKG, "csrc"),
                    os.path.join(ROOT, "tools", "taskmap_check.cu"), "-L", PKG, "-lslimb200",
                    "-o", str(exe)], check=True, capture_output=True)
    env = dict(os.environ, LD_LIBRARY_PATH=PKG + os.pathsep + os.environ.get("LD_LIBRARY_PATH", ""))
    out = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all orders valid" in out.stdout
