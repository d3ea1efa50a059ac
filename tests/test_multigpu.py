"""Multi-GPU parity (2/4/8 B200s of one box): halo exchange bit-exact vs the global periodic
wrap, P-GPU result bit-identical to 1 GPU, and oracle parity.  Skipped with fewer GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(nproc, N, corners=0, steps=3, port=29511, exchange="p2p", radius=3, dtype="f64"):
    env = dict(os.environ, MGPU_N=",".join(map(str, N)), MGPU_CORNERS=str(corners), MGPU_STEPS=str(steps),
               MGPU_EXCHANGE=exchange, MGPU_RADIUS=str(radius), MGPU_DTYPE=dtype)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tools", "mgpu_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("nproc", [2, 4, 8])
@pytest.mark.parametrize("corners", [0, 1])
@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_multigpu_halo_and_bit_identity(nproc, corners, exchange):
    """Both exchanges give the 1-GPU result bit for bit (so they agree with each other)."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    N = {2: (40, 36, 32), 4: (40, 32, 32), 8: (32, 32, 32)}[nproc]
    rc, out = _run(nproc, N, corners, port=29500 + nproc * 4 + corners * 2 + (exchange == "p2p"), exchange=exchange)
    assert rc == 0, out[-4000:]


@pytest.mark.parametrize("radius", [1, 2, 4])
def test_multigpu_other_orders(radius):
    """Orders 2, 4, 8 on 2 GPUs with the peer-memory exchange: bitwise halo, 1-vs-2 GPU identity."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    rc, out = _run(2, (40, 36, 32), 0, port=29560 + radius, exchange="p2p", radius=radius)
    assert rc == 0, out[-4000:]


@pytest.mark.parametrize("nproc,exchange", [(2, "p2p"), (4, "nccl"), (4, "p2p")])
def test_multigpu_fp32(nproc, exchange):
    """The FP32 variant: bitwise halo (FP32-exact sentinels), P-GPU = 1-GPU bit for bit, oracle
    within 1e-4 (R#18)."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    rc, out = _run(nproc, (40, 32, 32), 0, port=29570 + nproc * 2 + (exchange == "p2p"), exchange=exchange,
                   dtype="f32")
    assert rc == 0, out[-4000:]


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_multigpu_full_size_bit_identity(nproc):
    """BASELINE's 512^3 strong-scaling grid in bench.py's launch configuration (peer memory):
    every rank's state after one RK3 step equals the same region of a 1-GPU 512^3 run, bitwise."""
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, MGPU_N="512,512,512", MGPU_EXCHANGE="p2p")  # bench.py's default at every N
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={29580 + nproc}", os.path.join(ROOT, "tools", "mgpu_full.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]


def test_multigpu_1024_checksum_identity():
    """BASELINE configs[4] (1024^3 FP64) on 4 B200s in bench.py's configuration: every rank's state
    after one RK3 step has the same bit-sensitive checksums as the same block of a 1-GPU 1024^3 run
    (137 GB of mesh workspace on one GPU).  Long (host-side ICs of 68 GB): opt in with
    B2MHD_TEST_1024=1."""
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    if os.environ.get("B2MHD_TEST_1024") != "1":
        pytest.skip("opt in with B2MHD_TEST_1024=1 (profiles/r02/mgpu/full1024_4gpu_vs_1gpu.json)")
    env = dict(os.environ, MGPU_N="1024,1024,1024", MGPU_EXCHANGE="p2p", MGPU_CHECKSUM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port=29592", os.path.join(ROOT, "tools", "mgpu_full.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=3000)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
