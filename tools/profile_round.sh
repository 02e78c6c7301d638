# Profile one C2 step on the GPU box (single stream so ncu does not serialise a
# side-stream kernel):
#   1. the launch list (gpu__time_duration per launch, --clock-control none)
#   2. the SURVEY §8(d) counters per hot kernel (one launch each): DRAM / L2
#      bytes, L2 RED requests (backward atomics), shared-memory wavefronts,
#      bank conflicts and utilisation, pipe utilisation
#   3. one --set full capture per hot kernel (source-level stalls)
# usage: bash tools/profile_round.sh <tag>
TAG=${1:-r2}
export CSPLAT_SINGLE_STREAM=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py 3 > gpurun_out/prof_launch.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed
M=$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum
M=$M,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none --csv -k regex:"k_render_bwd|k_render_fwd|k_sort_tiles|k_project|k_chain|k_prune_onepass|k_rvq" \
    --log-file gpurun_out/counters_$TAG.csv python tools/prof_step.py 2 > gpurun_out/prof_counters.log 2>&1
for k in k_render_bwd k_render_fwd k_sort_tiles k_project k_chain k_prune_onepass; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/prof_$k python tools/prof_step.py 2 > gpurun_out/prof_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_rvq_chunked" -s 2 -c 2 \
    -o gpurun_out/prof_k_rvq python tools/prof_step.py 2 > gpurun_out/prof_k_rvq.log 2>&1
ls gpurun_out
