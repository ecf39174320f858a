"""Golden fixture for generate_threshold_schedule, made by the REFERENCE itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_threshold_golden.py

It trains the reference's session model exactly as its conftest does
(pkg/tests/conftest.py:15-23: gauss8, 2-64-64-2 silu, 5000 Adam iterations,
lr 1e-3, seed 42, 50-step posterior schedule), runs the reference's own
sequential sampler at seed 42, and stores the trained weights, that run's eps
records and x0, and the schedule the reference derives from it with tau 0.1 /
max_len 4 — which must equal the reference's FROZEN_TAU01_SCHEDULE
(pkg/tests/test_engines.py:43-46, asserted at :363-367).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PARASTEP_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import parastep.engines as E  # noqa: E402
from parastep.predictor import TrainConfig, train  # noqa: E402
from parastep.schedule import make_default_schedule  # noqa: E402

FROZEN_TAU01_SCHEDULE = [
    1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 2, 1, 1,
    1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 1,
]


def main() -> None:
    sched = make_default_schedule(50)
    w = train(TrainConfig(dataset="gauss8", hidden=(64, 64), iterations=5000,
                          learning_rate=1e-3, seed=42), sched)
    ref = E.run_strategy(w, sched, E.RunConfig(steps=50, strategy="sequential", seed=42,
                                               data_dim=w.data_dim))
    lengths = E.generate_threshold_schedule(ref, 0.1, 4)
    assert lengths == FROZEN_TAU01_SCHEDULE, lengths
    arrays = {"activation": np.array(w.activation), "n_layers": np.array(len(w.layers)),
              "ts": np.array([r.t for r in ref.records]),
              "eps": np.stack([r.eps for r in ref.records]),
              "xs": np.stack([r.x for r in ref.records]), "x0": ref.x0,
              "schedule_tau01_len4": np.array(lengths)}
    for i, layer in enumerate(w.layers):
        arrays[f"w{i}"] = layer.w
        arrays[f"b{i}"] = layer.b
    np.savez_compressed(os.path.join(HERE, "threshold_tau01.npz"), **arrays)
    print("wrote threshold_tau01.npz", lengths)


if __name__ == "__main__":
    main()
