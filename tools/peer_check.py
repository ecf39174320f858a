"""Peer-memory exchange check (launched by torchrun with --nproc-per-node P).

Each process runs ParaStep with degree = world size through NcclSampler with
exchange="peer" (CUDA IPC buffers + flag kernels; the bootstrap group is
gloo, no NCCL). With PEER_SAME_GPU=1 every rank uses cuda:0 - the way the
exchange protocol (IPC mapping, release/acquire flags, double buffering) is
exercised on a one-GPU box. Rank 0 compares the eager and graph-replayed
runs against the single-process lane emulation bit for bit; every rank's x0
must equal rank 0's. Prints "PEER_CHECK OK ..." on success.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2505_14741_b200 import engines as E, schedule as S  # noqa: E402
from paper_2505_14741_b200.dit import DiTWeights  # noqa: E402
from paper_2505_14741_b200.protocol import NcclSampler  # noqa: E402
from paper_2505_14741_b200.spec import SPECS  # noqa: E402


def dbg(*a):
    if os.environ.get("PEER_DEBUG"):
        print(f"[rank {os.environ.get('RANK')}]", *a, file=sys.stderr, flush=True)


def main():
    same = os.environ.get("PEER_SAME_GPU", "0") == "1"
    local = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dbg("pg up")
    spec = SPECS[os.environ.get("PEER_CHECK_SPEC", "dit_tiny")]
    w = DiTWeights(spec, seed=4, max_batch=max(2, world))
    T = int(os.environ.get("PEER_CHECK_T", "13"))  # 13 = 2 warm-up + cycles with a truncated tail
    sched = S.make_default_schedule(T)
    cfg = E.RunConfig(steps=T, warmup=2, strategy="parastep", degree=world, seed=7,
                      data_dim=spec.data_dim)
    dbg("weights built")
    s = NcclSampler(w, sched, cfg, record=True, exchange="peer")
    dbg("sampler built (ipc mapped)")
    s.run(7)
    dbg("eager run issued")
    res = s.result()
    dbg("eager run done")
    s.run(7, graph=True)
    s.run(7, graph=True)  # replay: epochs advance on device
    g = s.result()
    # measured exchange ledger of the peer reads + the device-clock phase split
    from paper_2505_14741_b200.ledger import verify_merged

    verify_merged(res.ledgers, E.plan_cycles(cfg))
    ts = NcclSampler(w, sched, cfg, record=False, exchange="peer", timed=True)
    ts.run(7)
    tr = ts.result()
    assert tr.loop_latency_s > 0 and np.array_equal(tr.x0, res.x0)
    ts.ops.px.close()
    x0s = [None] * world
    dist.all_gather_object(x0s, res.x0)
    ok = all(np.array_equal(x0s[0], v) for v in x0s) and np.array_equal(g.x0, res.x0)
    if rank == 0:
        ref = E.run_strategy(w, sched, cfg)  # lane emulation on one GPU
        ok = ok and res.trajectory.bitwise_equal(ref) and g.trajectory.bitwise_equal(ref)
        print(f"PEER_CHECK {'OK' if ok else 'FAIL'} world={world} same_gpu={same} "
              f"rounds={res.gathers} launches={res.launches} "
              f"loop_ms={tr.loop_latency_s * 1e3:.3f}", flush=True)
    dist.barrier()
    s.ops.px.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
