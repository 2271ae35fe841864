# Shared-memory / L2 / DRAM traffic counters of the hot kernels (one launch each, ncu replay):
# tensor-core operand reads (utcmma matrix A / B wavefronts), LSU shared loads/stores, bank
# reads/writes and their % of peak, TMA bytes into shared memory, L2 and DRAM bytes.
#   bash tools/ncu_smem.sh OUTDIR
OUT=${1:-gpurun_out}
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg
M=$M,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum
M=$M,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__data_pipe_tc_wavefronts.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum
M=$M,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum
M=$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
M=$M,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_red.sum
M=$M,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.sum
M=$M,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
for w in bwd fwd fwd128; do
  k=$([ $w = bwd ] && echo bwd_bf16 || ([ $w = fwd ] && echo fwd_db || echo fwd128))
  timeout 600 ncu --metrics $M --clock-control none -k regex:$k -s 1 -c 1 --csv python tools/prof_kernel.py $w > $OUT/ncu_smem_$w.csv 2> $OUT/ncu_smem_$w.err
  echo "ncu smem $w $?"
done
