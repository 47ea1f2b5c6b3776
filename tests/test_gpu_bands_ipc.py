"""The multi-process row-band layout on real CUDA-IPC mappings (SURVEY 8(e),
config C4 across GPUs): two processes, one band each, exchange their band
records over torch.distributed (gloo) and store halo rows into each other's
allocations from a kernel. Both processes share the one GPU of this
environment, which CUDA IPC allows; the persistent solve itself needs one
GPU per band (tests/test_gpu_bands.py runs it with every band in one launch)."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_two_process_band_halo_over_ipc(world):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port),
                        os.path.join(ROOT, "tests", "dist_bands_ipc_worker.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count('"checks"') == world
