"""B200-native ParaStep (arXiv 2505.14741): the reuse-then-predict denoise loop.

Drop-in for the reference package ``parastep`` on its hot path; modules mirror
the reference's names:

    numerics   counter RNG (GPU), rel_mae
    schedule   NoiseSchedule, make_default_schedule, ddpm_step (GPU)
    predictor  reference MLP: PredictorWeights, init_weights, forward, forward_batch
    dit        DiT-shaped predictors (BASELINE.json configs)
    engines    RunConfig, run_strategy, denoise_* , DeviceSampler (GPU)
    protocol   run_nccl: one process per GPU, one eps all-gather per round

Compute runs in the in-tree C-ABI library ``libparastep_b200.so`` (sm_100a);
there is no CPU fallback.
"""

__version__ = "0.1.0"
