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


def test_two_process_mailbox_exchange_bitwise():
    out = os.path.join(REPO, "gpurun_out", "ipc_two_ranks.txt")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if os.path.exists(out):
        os.remove(out)
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ipc_two_ranks.py"), "--same-gpu"],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    assert open(out).read().startswith("OK"), open(out).read()
