cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout -s KILL 600 python bench.py --config dit_xl2_bf16 --steps 3 --warmup 2 --batchstep 2 4 > gpurun_out/r2_bench_xl.json 2> gpurun_out/r2_bench_xl.err
timeout -s KILL 300 python bench.py --config c1ref_mlp --steps 5 --warmup 3 > gpurun_out/r2_bench_mlp.json 2> gpurun_out/r2_bench_mlp.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_dits2.csv python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r2_ncu1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 10 -c 2 -o gpurun_out/r2_gemm_fp32 python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r2_ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 5 -c 1 -o gpurun_out/r2_cycle python tools/profile_denoise.py --config small_dit_fp32 --degree 4 --strategy batchstep > gpurun_out/r2_ncu3.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_xl.csv python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r2_ncu4.log 2>&1
