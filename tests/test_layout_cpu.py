"""Host-side check of the fine factor plane layout (smoother.cuh plane_off /
diag_slot / mv_chunk_pos) for every build knob: tools/layout_check.cu is
compiled with nvcc and run on the host (no GPU)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

KNOBS = [("rows1", ["-DTMG_MV_ROWS=1"]), ("rows2", ["-DTMG_MV_ROWS=2"]),
         ("rows2_packed", ["-DTMG_MV_ROWS=2", "-DTMG_DIAG_PACK=1"]), ("rows4", ["-DTMG_MV_ROWS=4"])]


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not found")
@pytest.mark.parametrize("name,defs", KNOBS, ids=[k[0] for k in KNOBS])
def test_plane_layout(tmp_path, name, defs):
    exe = str(tmp_path / f"layout_{name}")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O0", "-std=c++17",
                           "--expt-relaxed-constexpr", *defs, "-I",
                           os.path.join(ROOT, "paper_2410_06850_b200", "csrc"),
                           os.path.join(ROOT, "tools", "layout_check.cu"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.count("bad=0") == 2, out.stdout
