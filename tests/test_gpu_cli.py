"""Operator CLI on the GPU: generate writes the reference's
files (trajectory.txt in the reference text format, samples.csv,
summary.txt) whose content matches the engine run; compare writes the
divergence tables from device-side diffs; generate over a torchrun NCCL
group writes the traffic census and checks it against the closed form."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2505_14741_b200 import cli, engines as E, predictor as P  # noqa: E402
from paper_2505_14741_b200 import schedule as S, trajectory_io as TIO  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generate_mlp_parastep(tmp_path):
    rc = cli.main(["generate", "--strategy", "parastep", "-p", "3", "--warmup", "2",
                   "--steps", "12", "--samples", "2", "--seed", "4", "--out-dir", str(tmp_path)])
    assert rc == 0
    tr = TIO.load_trajectory_text(tmp_path / "trajectory.txt")
    w = P.init_weights(P.TrainConfig(data_dim=2, hidden=(64, 64), embed_dim=16, seed=7,
                                     iterations=0))
    ref = E.run_strategy(w, S.make_default_schedule(12), E.RunConfig(
        steps=12, warmup=2, strategy="parastep", degree=3, seed=4, data_dim=2))
    assert tr.bitwise_equal(ref)
    rows = (tmp_path / "samples.csv").read_text().splitlines()
    assert rows[0] == "sample,x0,x1" and len(rows) == 3
    assert np.array_equal(np.array([float(v) for v in rows[1].split(",")[1:]]), ref.x0)
    summary = (tmp_path / "summary.txt").read_text()
    assert "fresh_calls=" in summary and "strategy=parastep" in summary


def test_compare_dit(tmp_path):
    rc = cli.main(["compare", "--predictor", "dit_tiny", "--strategies",
                   "parastep:2,direct_reuse:2", "--seeds", "2", "--steps", "10", "--warmup", "2",
                   "--out-dir", str(tmp_path)])
    assert rc == 0
    div = (tmp_path / "divergence.csv").read_text().splitlines()
    assert div[0] == "strategy,seed,final_rel_mae,final_mse" and len(div) == 5
    assert "win_rate=" in (tmp_path / "summary.txt").read_text()


def test_compare_files_match_reference_semantics(tmp_path):
    """adjacent.csv holds the strategy's OWN adjacent-step series (T-1 rows per
    run, reference cli.py:530-535) and divergence.csv the x0 MSE (not x_1's)."""
    steps, warm = 10, 2
    rc = cli.main(["compare", "--strategies", "sequential:1,parastep:3", "--seeds", "1",
                   "--steps", str(steps), "--warmup", str(warm), "--seed", "3",
                   "--out-dir", str(tmp_path)])
    assert rc == 0
    w = P.init_weights(P.TrainConfig(data_dim=2, hidden=(64, 64), embed_dim=16, seed=7,
                                     iterations=0))
    sch = S.make_default_schedule(steps, "posterior")
    seq = E.run_strategy(w, sch, E.RunConfig(steps=steps, seed=3, data_dim=2))
    par = E.run_strategy(w, sch, E.RunConfig(steps=steps, warmup=warm, strategy="parastep",
                                             degree=3, seed=3, data_dim=2))
    adj = (tmp_path / "adjacent.csv").read_text().splitlines()
    assert adj[0] == "strategy,seed,step,rel_mae_x,rel_mae_eps"
    assert len(adj) == 1 + 2 * (steps - 1)
    for label, tr, lines in (("sequential:1", seq, adj[1:steps]),
                             ("parastep:3", par, adj[steps:])):
        want = E.compare_trajectories(seq, tr).adjacent_b
        for line, r in zip(lines, want):
            lab, seed, t, rx, re_ = line.split(",")
            assert (lab, int(seed), int(t)) == (label, 3, r.t)
            assert np.isclose(float(rx), r.rel_mae_x, rtol=1e-10)
            assert np.isclose(float(re_), r.rel_mae_eps, rtol=1e-10)
    div = (tmp_path / "divergence.csv").read_text().splitlines()
    rep = E.compare_trajectories(seq, par)
    lab, seed, fr, fm = div[2].split(",")
    assert lab == "parastep:3"
    assert np.isclose(float(fr), rep.final_rel_mae, rtol=1e-10)
    assert np.isclose(float(fm), rep.final_mse, rtol=1e-10)
    assert float(div[1].split(",")[3]) == 0.0  # sequential vs itself


def test_generate_nccl_traffic_census(tmp_path):
    n = torch.cuda.device_count()
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
         "--master-addr", "127.0.0.1", "--master-port", "29731", "-m",
         "paper_2505_14741_b200.cli", "generate", "--backend", "nccl", "--strategy",
         "parastep", "-p", str(n), "--warmup", "2", "--steps", "12", "--predictor", "dit_tiny",
         "--out-dir", str(tmp_path)],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    summary = (tmp_path / "summary.txt").read_text()
    assert "traffic=ok" in summary
    lines = (tmp_path / "traffic.csv").read_text().splitlines()
    assert lines[0] == "round,cycle_len,sent_bytes,received_bytes"
