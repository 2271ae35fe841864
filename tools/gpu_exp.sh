set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_single_query.py tests/test_gpu_partial.py -x -q > gpurun_out/t_sq.log 2>&1; tail -n 2 gpurun_out/t_sq.log
timeout 300 python tools/sq_pool.py gpurun_out/sq_pool2.json > gpurun_out/sq_pool2.log 2>&1
timeout 300 python tools/sq_timeline.py > gpurun_out/sq_timeline2.log 2>&1
bash tools/ncu_smem.sh gpurun_out
