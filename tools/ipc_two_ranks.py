"""Two processes, one mailbox-connected rank plan each (CUDA IPC), on one GPU or two.

    python tools/ipc_two_ranks.py [--same-gpu] [--stuck-rank R | --kill-rank R]

Each rank owns its octant range of the volume; roots are exchanged by the
loop kernels through each other's mailboxes.  Rank 0 compares the result with
a single-process solve bit for bit.  (On one GPU the two cooperative kernels
time-share the device; the in-kernel exchange has a 4 s timeout.)

Failure modes: with --stuck-rank R, rank R connects its mailbox and then never
runs (a hung peer); with --kill-rank R it exits right after connecting (a
crashed peer).  The other rank runs with a 300 ms peer timeout and must fail
with FCM_E_NCCL (DeviceError) naming rank R and the pass it waited for.
"""
import os
import sys

import numpy as np
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, same_gpu, out, stuck=-1, kill=-1):
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import torch
    import torch.distributed as dist
    import paper_1601_00072_b200 as pkg
    from paper_1601_00072_b200 import _lib
    from conftest import mixture_pixels
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = int(os.environ.get("FCM_IPC_N", "300007"))  # (> 8.4 M voxels: >1024 tiles per rank, owner path)
    x = np.clip(np.rint(mixture_pixels(n, 3, seed=9)), 0, 255).astype(np.uint8)
    dev = 0 if same_gpu else rank
    plan = pkg.FcmPlan.for_rank(n, 3, _lib.FCM_X_U8, dev, world, rank, None)
    plan.upload_pixels(x[plan.voxel0:plan.voxel0 + plan.n_local])
    plan.init_membership(4)
    mine = torch.frombuffer(bytearray(plan.mailbox_handle()), dtype=torch.uint8)
    allh = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allh, mine)
    plan.connect_peers(b"".join(bytes(t.numpy().tobytes()) for t in allh), world)
    dist.barrier()
    if kill == rank:
        os._exit(0)  # a crashed peer: no run, no goodbye
    if stuck >= 0 or kill >= 0:
        bad = stuck if stuck >= 0 else kill
        if rank == bad:  # a hung peer: alive, mailbox mapped, never runs
            dist.barrier()
        else:
            plan.set_option(_lib.FCM_OPT_PEER_TIMEOUT_MS, 300)
            try:
                plan.run(2.0, 1e-5, 100)
                msg = "NO-ERROR"
            except pkg.DeviceError as e:
                msg = f"OK-FAILED {e}" if f"of rank {bad} " in str(e) else f"WRONG-RANK {e}"
            except Exception as e:  # noqa: BLE001
                msg = f"WRONG-ERROR {type(e).__name__}: {e}"
            with open(out, "w") as f:
                f.write(msg + "\n")
            if stuck >= 0:
                dist.barrier()
        plan.close()
        if stuck >= 0:
            dist.destroy_process_group()
        return
    v, trace, k, conv = plan.run(2.0, 1e-5, 100)
    u, lab = plan.download()
    parts = [None] * world
    dist.all_gather_object(parts, (plan.voxel0, u.tobytes(), lab.tobytes()))
    if rank == 0:
        with pkg.FcmPlan(n, 3, _lib.FCM_X_U8, devices=[0]) as ref:
            ref.upload_pixels(x)
            ref.init_membership(4)
            rv, rt, rk, rc = ref.run(2.0, 1e-5, 100)
            ru, rl = ref.download()
        u_all = b"".join(p[1] for p in sorted(parts))
        l_all = b"".join(p[2] for p in sorted(parts))
        ok = (rk == k and v.tobytes() == rv.tobytes() and trace.tobytes() == rt.tobytes()
              and u_all == ru.tobytes() and l_all == rl.tobytes())
        with open(out, "w") as f:
            f.write(f"{'OK' if ok else 'MISMATCH'} iters={k} v={v}\n")
    plan.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    same = "--same-gpu" in sys.argv
    stuck = int(sys.argv[sys.argv.index("--stuck-rank") + 1]) if "--stuck-rank" in sys.argv else -1
    kill = int(sys.argv[sys.argv.index("--kill-rank") + 1]) if "--kill-rank" in sys.argv else -1
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = os.path.join(REPO, "gpurun_out", "ipc_two_ranks.txt")
    mp.spawn(worker, args=(2, port, same, out, stuck, kill), nprocs=2, join=True)
    print(open(out).read())
