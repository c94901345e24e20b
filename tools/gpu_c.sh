mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"; cat gpurun_out/bench_c.json; tail -3 gpurun_out/bench_c.err
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_tma -c 1 -o gpurun_out/gemm_tma -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_wgrad_tma -s 2 -c 1 -o gpurun_out/wgrad_tma -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu2 rc=$?"
