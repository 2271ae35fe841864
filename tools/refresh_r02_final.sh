# Round-2 measurement refresh (run on the GPU box from the repo root): GPU tests, smoke, the
# bench line, the headline-step launch list, and ncu --set full captures of the hot kernels.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_r02.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/t_r02.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; echo "smoke $?"
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_step_r02.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/ncu_step_r02.log 2>&1; echo "ncu step $?"
for w in fwd:fwd_db bwd:bwd_bf16 sq:sq_bf16 sq_batch:sq_bf16 fwd128:fwd128 bwd128:bwd128; do
  what=${w%%:*}; kern=${w##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s 1 -c 1 -f -o gpurun_out/prof_${what}_r02 python tools/prof_kernel.py $what > gpurun_out/ncu_${what}_r02.log 2>&1; echo "ncu $what $?"
done
