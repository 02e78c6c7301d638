# Profile one C2 step on the GPU box: launch list + one --set full capture per
# hot kernel (single stream so ncu does not serialise a side-stream kernel).
# usage: bash tools/profile_round.sh <tag>
TAG=${1:-r1}
export CSPLAT_SINGLE_STREAM=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py 3 > gpurun_out/prof_launch.log 2>&1
for k in k_render_bwd k_render_fwd k_sort_tiles k_project k_chain k_prune_onepass; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/prof_$k python tools/prof_step.py 2 > gpurun_out/prof_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"k_rvq_chunked" -s 2 -c 2 \
    -o gpurun_out/prof_k_rvq python tools/prof_step.py 2 > gpurun_out/prof_k_rvq.log 2>&1
ls gpurun_out
