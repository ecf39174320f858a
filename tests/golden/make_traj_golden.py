"""Reference-written trajectory files (trajectory_io.py formats) for the
format-parity tests. Run in the build container only (needs /root/reference):

    python tests/golden/make_traj_golden.py

The reference's tiny_w (tests/conftest.py:44-53) runs ParaStep p=3 through
its own engine and saves the result with its own ``save_trajectory_text`` /
``save_trajectory_binary``.
"""

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("PARASTEP_REF_SRC", "/root/reference/pkg/src"))

import parastep.engines as E  # noqa: E402
from parastep.predictor import TrainConfig, init_weights  # noqa: E402
from parastep.schedule import make_default_schedule  # noqa: E402
from parastep.trajectory_io import save_trajectory_binary, save_trajectory_text  # noqa: E402

w = init_weights(TrainConfig(hidden=(8,), embed_dim=4, seed=7, activation="silu", iterations=0))
cfg = E.RunConfig(steps=12, warmup=4, strategy="parastep", degree=3, seed=5, data_dim=2)
tr = E.run_strategy(w, make_default_schedule(12), cfg)
save_trajectory_text(tr, os.path.join(HERE, "traj_ps3.txt"))
save_trajectory_binary(tr, os.path.join(HERE, "traj_ps3.pstj"))
print("wrote traj_ps3.txt / traj_ps3.pstj")
