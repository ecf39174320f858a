cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py tests/test_gpu_sampler.py -q -x 2>&1 | tail -15 > gpurun_out/r3_tests.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
timeout -s KILL 600 python bench.py --config dit_xl2_bf16 --steps 3 --warmup 2 --batchstep 4 --no-cpu-baseline > gpurun_out/r3_bench_xl.json 2> gpurun_out/r3_bench_xl.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_dits2.csv python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r3_ncu1.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_xl.csv python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r3_ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 4 -o gpurun_out/r3_gemm_xl python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r3_ncu3.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 4 -o gpurun_out/r3_gemm_s2 python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r3_ncu4.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn|gemv|ln_mod" -s 30 -c 6 -o gpurun_out/r3_misc_xl python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r3_ncu5.log 2>&1
