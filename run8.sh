cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 300 python tools/gemm_probe.py > gpurun_out/r8_probe.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py tests/test_gpu_sampler.py -q -x 2>&1 | tail -15 > gpurun_out/r8_tests.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err
timeout -s KILL 600 python bench.py --config dit_xl2_bf16 --steps 3 --warmup 2 --batchstep 4 8 --no-cpu-baseline > gpurun_out/r8_bench_xl.json 2> gpurun_out/r8_bench_xl.err
