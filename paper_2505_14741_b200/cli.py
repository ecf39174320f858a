"""Operator surface: ``python -m paper_2505_14741_b200.cli generate|compare``
(the reference's cmd_generate / cmd_compare,
pkg/src/parastep/cli.py:379-575, same outputs and exit codes).

generate  one or more samples with any strategy, on one GPU (DeviceSampler:
          the d lanes of ParaStep run as lanes of one device) or, under
          ``torchrun --nproc-per-node d``, one rank per GPU over NCCL
          (``--backend nccl``). Writes trajectory.txt (the reference's text
          format), samples.csv, summary.txt; the NCCL backend adds
          traffic.csv, the per-round all-gather census checked against its
          closed form (each rank sends N*s and receives (d-1)*N*s bytes per
          full round; the reference's Algorithm-1 ledger moves 2(d-1)*M per
          cycle, protocol/ledger.py:120-123).
compare   strategies against the sequential reference over seeds, with the
          per-step divergence computed on device (ps_traj_diff); writes
          adjacent.csv, divergence.csv, summary.txt.

Predictors: ``--predictor mlp`` is the reference's MLP (init_weights, fp64),
the others are the BASELINE.json network shapes (random init, reference
Xavier convention). Exit codes: 2 for configuration / parameter errors, 3
for other package or OS errors (cli.py:727-736).
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys
from pathlib import Path

from .engines import (
    STRATEGIES,
    STRATEGY_DIRECT_REUSE,
    STRATEGY_DYNAMIC,
    STRATEGY_PARASTEP,
    STRATEGY_SEQUENTIAL,
    DeviceSampler,
    RunConfig,
    compare_trajectories_device,
    warmup_from_ratio,
)
from .errors import ConfigError, ParameterError, ParastepError
from .schedule import make_default_schedule
from .trajectory_io import save_trajectory_text

PREDICTORS = ("mlp", "dit_tiny", "dit_s2", "dit_xl2", "cogvideox_2b", "unet_tiny",
              "audioldm2_large")


def _f(v: float) -> str:
    return repr(float(v))


def _weights(ns):
    from . import predictor as P

    name = ns.predictor
    if name == "mlp":
        return P.init_weights(P.TrainConfig(data_dim=ns.data_dim or 2, hidden=(64, 64),
                                            embed_dim=16, seed=ns.weight_seed, iterations=0))
    if name.startswith("unet") or name.startswith("audioldm"):
        from .unet import UNetWeights

        return UNetWeights(name, seed=ns.weight_seed, max_batch=max(ns.degree, 1))
    from .dit import DiTWeights

    return DiTWeights(name, seed=ns.weight_seed, precision=ns.precision,
                      max_batch=max(ns.degree, 1))


def _warmup(ns) -> int:
    if ns.warmup is not None and ns.warmup_ratio is not None:
        raise ConfigError("give --warmup or --warmup-ratio, not both")
    if ns.warmup_ratio is not None:
        return warmup_from_ratio(ns.warmup_ratio, ns.steps)
    return ns.warmup if ns.warmup is not None else 0


def _cfg(ns, w, seed, warmup, strategy=None, degree=None):
    lengths = None
    strategy = strategy or ns.strategy
    if strategy == STRATEGY_DYNAMIC:
        if not ns.cycle_lengths:
            raise ConfigError("dynamic strategy needs --cycle-lengths")
        lengths = [int(v) for v in ns.cycle_lengths.split(",")]
    return RunConfig(steps=ns.steps, warmup=warmup, strategy=strategy,
                     degree=degree if degree is not None else ns.degree,
                     schedule_override=lengths, seed=seed, data_dim=w.data_dim)


def _out(ns) -> Path:
    d = Path(ns.out_dir or ".")
    d.mkdir(parents=True, exist_ok=True)
    return d


def cmd_generate(ns) -> int:
    if ns.samples < 1:
        raise ConfigError(f"samples must be >= 1, got {ns.samples}")
    warmup = _warmup(ns)
    sched = make_default_schedule(ns.steps, ns.sigma_mode)
    w = _weights(ns)
    out = _out(ns)
    nccl = ns.backend == "nccl"
    rank, world = 0, 1
    if nccl:
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        rank, world = dist.get_rank(), dist.get_world_size()
        if ns.strategy != STRATEGY_PARASTEP or ns.degree != world:
            raise ConfigError("--backend nccl runs parastep with degree == world size")
    finals, first, census = [], None, None
    for i in range(ns.samples):
        cfg = _cfg(ns, w, ns.seed + i, warmup)
        if nccl:
            from .protocol import NcclSampler

            s = NcclSampler(w, sched, cfg, record=True)
            traj = s.sample(cfg.seed)
            if i == 0:
                census = s.traffic_census()
        else:
            s = DeviceSampler(w, sched, cfg, record=True)
            traj = s.sample(cfg.seed)
        if rank != 0:
            continue
        if i == 0:
            first = traj
            save_trajectory_text(traj, out / "trajectory.txt")
        finals.append(traj.x0)
    if rank != 0:
        return 0
    rows = ["sample," + ",".join(f"x{j}" for j in range(w.data_dim))]
    rows += [f"{i}," + ",".join(_f(v) for v in x0) for i, x0 in enumerate(finals)]
    (out / "samples.csv").write_text("\n".join(rows) + "\n")
    summary = ["command=generate", f"strategy={ns.strategy}", f"degree={ns.degree}",
               f"steps={ns.steps}", f"warmup={warmup}", f"sigma_mode={ns.sigma_mode}",
               f"samples={ns.samples}", f"predictor={ns.predictor}",
               f"fresh_calls={first.fresh_calls}", f"batch_calls={first.batch_calls}",
               f"backend={ns.backend}"]
    if census is not None:
        (out / "traffic.csv").write_text(census["csv"])
        summary += [f"allgathers={census['rounds']}", f"sent_bytes={census['sent']}",
                    f"received_bytes={census['received']}",
                    f"traffic={'ok' if census['ok'] else 'MISMATCH'}"]
    (out / "summary.txt").write_text("\n".join(summary) + "\n")
    print("\n".join(summary))
    print(f"wrote {out / 'trajectory.txt'}, {out / 'samples.csv'}")
    return 0


def cmd_compare(ns) -> int:
    if not ns.strategies:
        raise ConfigError("at least one strategy spec is required (--strategies name[:degree])")
    specs = []
    for item in ns.strategies.split(","):
        name, colon, deg = item.partition(":")
        if name not in STRATEGIES:
            raise ConfigError(f"strategies: unknown strategy {name!r}; one of {', '.join(STRATEGIES)}")
        d = int(deg) if colon else 1
        if d < 1:
            raise ConfigError(f"strategies: degree must be >= 1 in {item!r}")
        specs.append((name, d))
    if ns.seeds < 1:
        raise ConfigError(f"seeds must be >= 1, got {ns.seeds}")
    warmup = _warmup(ns)
    sched = make_default_schedule(ns.steps, ns.sigma_mode)
    ns.degree = max(d for _, d in specs)
    w = _weights(ns)
    out = _out(ns)
    adjacent = ["strategy,seed,step,rel_mae_x,rel_mae_eps"]
    divergence = ["strategy,seed,final_rel_mae,final_mse"]
    finals: dict[str, list[float]] = {}
    refs = []
    for i in range(ns.seeds):
        r = DeviceSampler(w, sched, _cfg(ns, w, ns.seed + i, 0, STRATEGY_SEQUENTIAL, 1))
        r.run(ns.seed + i)
        refs.append(r)
    for name, d in specs:
        label = f"{name}:{d}"
        finals[label] = []
        for i in range(ns.seeds):
            if name == STRATEGY_SEQUENTIAL:
                s = refs[i]
            else:
                s = DeviceSampler(w, sched, _cfg(ns, w, ns.seed + i, warmup, name, d))
                s.run(ns.seed + i)
            report = compare_trajectories_device(refs[i], s)
            # the strategy's own adjacent-step series (T-1 rows, cli.py:530-535)
            adjacent += [f"{label},{ns.seed + i},{r.t},{_f(r.rel_mae_x)},{_f(r.rel_mae_eps)}"
                         for r in report.adjacent_b]
            divergence.append(f"{label},{ns.seed + i},{_f(report.final_rel_mae)},"
                              f"{_f(report.final_mse)}")
            finals[label].append(report.final_rel_mae)
    (out / "adjacent.csv").write_text("\n".join(adjacent) + "\n")
    (out / "divergence.csv").write_text("\n".join(divergence) + "\n")
    summary = ["command=compare", f"seeds={ns.seeds}", f"steps={ns.steps}", f"warmup={warmup}"]
    for label, v in finals.items():
        summary.append(f"strategy={label} mean_final_rel_mae={statistics.mean(v):.6g} "
                       f"median_final_rel_mae={statistics.median(v):.6g}")
    para = next((f"{n}:{d}" for n, d in specs if n == STRATEGY_PARASTEP), None)
    reuse = next((f"{n}:{d}" for n, d in specs if n == STRATEGY_DIRECT_REUSE), None)
    if para and reuse:
        wins = sum(1 for a, b in zip(finals[para], finals[reuse]) if a < b)
        summary.append(f"win_rate={wins / ns.seeds:.4f} ({wins}/{ns.seeds}) {para} vs {reuse}")
    else:
        summary.append("win_rate=n/a")
    (out / "summary.txt").write_text("\n".join(summary) + "\n")
    print("\n".join(summary))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2505_14741_b200.cli")
    sub = ap.add_subparsers(dest="command", required=True)
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--seed", type=int, default=0)
    common.add_argument("--out-dir", dest="out_dir")
    common.add_argument("--steps", type=int, default=50)
    common.add_argument("--sigma-mode", dest="sigma_mode", choices=("posterior", "zero"),
                        default="posterior")
    common.add_argument("--warmup", type=int)
    common.add_argument("--warmup-ratio", dest="warmup_ratio", type=float)
    common.add_argument("--predictor", choices=PREDICTORS, default="mlp")
    common.add_argument("--precision", choices=("fp32", "bf16"), default="fp32")
    common.add_argument("--weight-seed", dest="weight_seed", type=int, default=7)
    common.add_argument("--data-dim", dest="data_dim", type=int)
    g = sub.add_parser("generate", parents=[common], help="sample with one strategy")
    g.add_argument("--strategy", choices=STRATEGIES, default=STRATEGY_SEQUENTIAL)
    g.add_argument("-p", "--degree", dest="degree", type=int, default=1)
    g.add_argument("--samples", type=int, default=1)
    g.add_argument("--cycle-lengths", dest="cycle_lengths")
    g.add_argument("--backend", choices=("device", "nccl"), default="device")
    g.set_defaults(func=cmd_generate)
    c = sub.add_parser("compare", parents=[common], help="strategies vs sequential")
    c.add_argument("--strategies")
    c.add_argument("--seeds", type=int, default=50)
    c.add_argument("--cycle-lengths", dest="cycle_lengths")
    c.set_defaults(func=cmd_compare, degree=1)
    return ap


def main(argv: list[str] | None = None) -> int:
    try:
        ns = build_parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return ns.func(ns)
    except (ConfigError, ParameterError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (ParastepError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
