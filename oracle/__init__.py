"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the ParaStep hot path.

This package is a from-text CPU restatement (numpy float64) of the reference
algorithm on the north-star path, written so the parity tests have an
independent checker for the CUDA product path:

- ``oracle.core``    counter-based RNG, schedule tables, ``ddpm_step``, the
                     reference MLP predictor and ``rel_mae``
                     (reference: pkg/src/parastep/numerics.py, schedule.py,
                     predictor.py)
- ``oracle.dit``     the DiT-shaped noise predictor restated in numpy
                     (no reference exists: parity for the DiT arithmetic is
                     pinned only through the reference *sampler* driving this
                     predictor via its import seam)
- ``oracle.engines`` sequential / direct-reuse / ParaStep (Algorithm 1,
                     virtual ranks) / cycle runner (BatchStep, dynamic)
                     (reference: pkg/src/parastep/engines.py)

Pinning: ``tests/golden/*.npz`` are produced by ``tests/golden/make_golden.py``
by importing the reference package itself (this container only) and running
its own functions; ``tests/test_oracle_golden.py`` checks this oracle against
every fixture bit-for-bit.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package ``paper_2505_14741_b200`` never
imports it.
"""
