set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_d128.py -x -q > gpurun_out/t_d128.log 2>&1; tail -n 15 gpurun_out/t_d128.log
timeout 600 python -m pytest tests/test_gpu_causal.py tests/test_gpu_padding.py tests/test_gpu_backward.py tests/test_gpu_fuzz.py tests/test_gpu_guard.py -x -q > gpurun_out/t_bwd.log 2>&1; tail -n 15 gpurun_out/t_bwd.log
CASE=bwd128 ITERS=10 timeout 300 python tools/ab.py paper_2112_05682_b200/libmea.so exp_so/exp_base.so > gpurun_out/ab_bwd128_fused.log 2>&1
