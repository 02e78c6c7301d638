export CSPLAT_SINGLE_STREAM=1
for k in k_bucket k_project k_sort_tiles k_render_bwd; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/p1_$k python tools/prof_step.py 2 > gpurun_out/p1_$k.log 2>&1
done
ls gpurun_out
