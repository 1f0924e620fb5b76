"""Multi-process fused exchange on one B200: two rank plans in two processes
(torch.distributed gloo only hands the 64-byte CUDA IPC handles around),
each running the whole solve in its loop kernel and writing its 2c+2 roots
into the other's mailbox every pass.  Rank 0 checks the result against a
single-process solve bit for bit (tools/ipc_two_ranks.py)."""

import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [300_007, 20_000_003])
def test_two_process_mailbox_exchange_bitwise(n):
    """300 K voxels: every CTA reduces the tile partials (small-volume pass
    end); 20 M voxels: 1,221 tiles per rank, level-1 owners and the
    seeded start inside each rank's loop kernel (pass 0 exchanges its root
    like every pass)."""
    out = os.path.join(REPO, "gpurun_out", "ipc_two_ranks.txt")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if os.path.exists(out):
        os.remove(out)
    env = dict(os.environ, FCM_IPC_N=str(n))
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ipc_two_ranks.py"), "--same-gpu"],
                       capture_output=True, text=True, timeout=400, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert open(out).read().startswith("OK"), open(out).read()


@pytest.mark.parametrize("mode", ["--stuck-rank", "--kill-rank"])
def test_dead_or_stuck_peer_names_the_rank(mode):
    """A peer that never publishes its per-pass root -- hung (alive, never
    runs) or crashed (exits after connecting) -- fails the surviving rank's
    fcm_run with FCM_E_NCCL (DeviceError) naming rank 1 and the pass, after
    the configured peer timeout (FCM_OPT_PEER_TIMEOUT_MS), instead of a 4 s
    spin ending in a generic internal error."""
    out = os.path.join(REPO, "gpurun_out", "ipc_two_ranks.txt")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if os.path.exists(out):
        os.remove(out)
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ipc_two_ranks.py"), "--same-gpu", mode, "1"],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    got = open(out).read()
    assert got.startswith("OK-FAILED"), got
    assert "rank 1" in got and "pass" in got
