"""NCCL path check on whatever GPUs are present (launched by torchrun).

Every rank runs ParaStep with degree = world size through ``run_nccl`` (eager)
and through ``NcclSampler`` with CUDA-graph capture (NCCL all-gathers inside
the graph); rank 0 compares both against the single-process lane emulation
(``run_strategy(parastep)``), which must be bit-identical, and every rank's
x0 must equal rank 0's. Prints one line "NCCL_CHECK OK ..." on success.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2505_14741_b200 import engines as E, schedule as S  # noqa: E402
from paper_2505_14741_b200.dit import DiTWeights  # noqa: E402
from paper_2505_14741_b200.protocol import NcclSampler, run_nccl  # noqa: E402
from paper_2505_14741_b200.spec import SPECS  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    spec = SPECS[os.environ.get("NCCL_CHECK_SPEC", "dit_tiny")]
    w = DiTWeights(spec, seed=4, max_batch=max(2, world))
    T = 16
    sched = S.make_default_schedule(T)
    cfg = E.RunConfig(steps=T, warmup=2, strategy="parastep", degree=world, seed=7,
                      data_dim=spec.data_dim)
    res = run_nccl(w, sched, cfg)
    # measured exchange ledger (raises LedgerViolationError on a mismatch) and
    # the per-rank device-clock split
    from paper_2505_14741_b200.ledger import verify_merged

    verify_merged(res.ledgers, E.plan_cycles(cfg))
    assert len(res.timings) == world and res.loop_latency_s > 0
    assert all(t.forward_s > 0 and t.apply_s > 0 for t in res.timings)
    # dynamic cycle lengths over the same rank loop (cycles <= world lanes)
    dyn_len = [min(world, 2), 1] * 8
    acc, lens = 0, []
    for c in dyn_len:
        if acc + c > T - 2:
            c = T - 2 - acc
        if c > 0:
            lens.append(c)
            acc += c
    dcfg = E.RunConfig(steps=T, warmup=2, strategy="dynamic", degree=world, seed=7,
                       schedule_override=lens, data_dim=spec.data_dim)
    dres = run_nccl(w, sched, dcfg)
    verify_merged(dres.ledgers, E.plan_cycles(dcfg))
    s = NcclSampler(w, sched, cfg, record=False)
    s.run(7, graph=True)
    s.run(7, graph=True)  # replay
    g = s.result()
    x0s = [torch.zeros(spec.data_dim, dtype=torch.float64, device="cuda") for _ in range(world)]
    dist.all_gather(x0s, torch.as_tensor(res.x0, device="cuda"))
    ok = all(torch.equal(x0s[0], v) for v in x0s) and np.array_equal(g.x0, res.x0)
    if rank == 0:
        ref = E.run_strategy(w, sched, cfg)  # lane emulation on one GPU
        ok = ok and res.trajectory.bitwise_equal(ref)
        dref = E.run_strategy(w, sched, dcfg)
        ok = ok and dres.trajectory.bitwise_equal(dref)
        t0 = res.timings[0]
        print(f"NCCL_CHECK {'OK' if ok else 'FAIL'} world={world} gathers={res.gathers} "
              f"launches={res.launches} loop_ms={res.loop_latency_s * 1e3:.3f} "
              f"fwd_ms={t0.forward_s * 1e3:.3f} xchg_ms={t0.exchange_wait_s * 1e3:.3f} "
              f"apply_ms={t0.apply_s * 1e3:.3f} ledger={res.ledgers[0].received}B", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
