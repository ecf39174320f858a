cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/r9_bench_default.json 2> gpurun_out/r9_bench_default.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches_dits2.csv python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r9_ncu1.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches_xl.csv python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r9_ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 4 -o gpurun_out/r9_gemm_dits2 python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r9_ncu3.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn_tc|ln_mod|cycle_kernel|gemv" -s 4 -c 4 -o gpurun_out/r9_misc_dits2 python tools/profile_denoise.py --config small_dit_fp32 > gpurun_out/r9_ncu4.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 4 -o gpurun_out/r9_gemm_xl python tools/profile_denoise.py --config dit_xl2_bf16 > gpurun_out/r9_ncu5.log 2>&1
timeout -s KILL 900 python bench.py --config cogvideox_bf16 --steps 3 --warmup 3 --batchstep --no-cpu-baseline > gpurun_out/r9_bench_cog.json 2> gpurun_out/r9_bench_cog.err
