"""The NCCL data plane of the library on >= 2 GPUs: one process per GPU via
torch.distributed.run, each driving its z-slab through dg_halo_exchange / ncclSend+Recv with the
interior/boundary overlap and ncclAllReduce (tests/_nccl_ranks.py).  Skipped on single-GPU
machines — the pool this repo is tested on gives one GPU per call, where the same multi-slab
layer is covered by the caller-transport loopback (test_gpu_slab_transport.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nproc", [2, 4])
def test_nccl_slabs_match_single_rank(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "_nccl_ranks.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=os.path.dirname(HERE))
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-3000:] + r.stderr[-5000:]
