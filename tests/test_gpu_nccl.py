"""Real multi-process parity (NCCL world over NVLink): every compressor x routine
pair and a mixed esp_sync_many strategy, one process per GPU (SURVEY.md 4
layer 4).  Needs >= 2 GPUs; runs under `gpurun --gpus 2|4`."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc", [1, 2, 4, 8])
def test_nccl_world_parity(nproc):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs, found {torch.cuda.device_count()}")
    import __graft_entry__
    __graft_entry__.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + nproc}",
           os.path.join(ROOT, "tests", "nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    assert r.stdout.count("sync_many ok") == nproc


@pytest.mark.parametrize("nproc", [1, 2, 4])
def test_ddp_comm_hook(nproc):
    """NEXT-4: the libesp DDP communication hook (paper_2205_14465_b200/ddp.py);
    one rank on a 1-GPU box (DDP still runs its reducer and the hook)."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs, found {torch.cuda.device_count()}")
    import __graft_entry__
    __graft_entry__.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}",
           os.path.join(ROOT, "tests", "ddp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    assert r.stdout.count("ddp hook ok") == nproc
