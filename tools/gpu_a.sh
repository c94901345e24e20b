mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_tma.log 2>&1; echo "gemm rc=$?"; tail -30 gpurun_out/gemm_tma.log
for spec in "c2:sage:hot=0.2:n=1:epochs=1" "c2:sage:hot=0.2:n=1:epochs=1" "c2:sage:hot=0.2:n=1:epochs=1:exec=serial" ; do
  HG_GEMM_LEGACY=1 timeout 600 python bench.py --epoch-mode "$spec" > gpurun_out/rep.log 2>&1; echo "$spec rc=$?"; grep -E "Error|error" gpurun_out/rep.log | head -3
done
CUDA_LAUNCH_BLOCKING=1 HG_GEMM_LEGACY=1 timeout 900 python bench.py --epoch-mode "c2:sage:hot=0.2:n=1:epochs=1:graph=0" > gpurun_out/rep_eager.log 2>&1; echo "eager rc=$?"; grep -B30 -E "Error" gpurun_out/rep_eager.log | grep -v "^frame" | head -60
