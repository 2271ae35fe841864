# Round-end measurement refresh (run on the GPU box from the repo root):
#   tests, the bench line, a 1-rank torchrun bench, the launch list and full ncu captures.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/t.log
timeout 600 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo "bench $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "torchrun $?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_launch.log 2>&1; echo "plain $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_step_r01.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/ncu_step.log 2>&1; echo "ncu step $?"
for w in fwd bwd sq fwd128; do
  timeout 300 python tools/prof_kernel.py $w > gpurun_out/plain_$w.log 2>&1; echo "plain $w $?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_db -s 1 -c 1 -f -o gpurun_out/prof_fwd_r01 python tools/prof_kernel.py fwd > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_bf16 -s 1 -c 1 -f -o gpurun_out/prof_bwd_r01 python tools/prof_kernel.py bwd > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sq_partial -s 1 -c 1 -f -o gpurun_out/prof_sq_r01 python tools/prof_kernel.py sq > gpurun_out/ncu_sq.log 2>&1; echo "ncu sq $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd128 -s 1 -c 1 -f -o gpurun_out/prof_fwd128_r01 python tools/prof_kernel.py fwd128 > gpurun_out/ncu_fwd128.log 2>&1; echo "ncu fwd128 $?"
for w in fwd bwd fwd128; do timeout 60 python tools/power_probe.py $w 5; done > gpurun_out/power.txt 2>&1; echo "power $?"
timeout 900 python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep $?"
timeout 900 python tools/paper_tables.py --out gpurun_out/paper_tables.json > gpurun_out/paper_tables.log 2>&1; echo "tables $?"
