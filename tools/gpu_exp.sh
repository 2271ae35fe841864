set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_forward.py -x -q -k "f32" > gpurun_out/t_f32.log 2>&1; tail -n 15 gpurun_out/t_f32.log
timeout 300 python tools/time_f32.py > gpurun_out/time_f32.log 2>&1; tail -n 5 gpurun_out/time_f32.log
