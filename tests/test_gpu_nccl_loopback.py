"""libmfx's NCCL transport on thread-ranks of one GPU through a loopback NCCL
stand-in (tests/nccl_loopback/: test infrastructure, MFX_NCCL_PATH).  Real NCCL
refuses two ranks on one device, so this is how the NCCL branches of the
exchange (GATHER send/recv groups, BCAST -- four grouped or one packed --,
the PSLAB gather, the multi-GPU p' halo exchange and dot all-gathers, and a
ncclCommSplit sub-communicator for a P-list subset) run on device buffers in
this environment.  Every case must reproduce the single-rank iteration
bitwise."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.join(ROOT, "tests", "nccl_loopback")
pytestmark = pytest.mark.gpu


def build_shim(tmpdir):
    out = os.path.join(tmpdir, "libnccl_loopback.so")
    cuda = "/usr/local/cuda"
    subprocess.check_call(["g++", "-shared", "-fPIC", "-O2", "-std=c++17", f"-I{cuda}/include",
                           os.path.join(HERE, "nccl_loopback.cpp"), "-o", out, f"-L{cuda}/lib64",
                           "-lcudart_static", "-lpthread", "-ldl", "-lrt"])
    return out


def test_nccl_transport_loopback(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    so = build_shim(str(tmp_path))
    r = subprocess.run([sys.executable, os.path.join(HERE, "run_loopback.py"), so], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "LOOPBACK OK" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
