# A/B library variants (tools/variants.py; "base" = in-tree) through bench.py:
# C2 step, stage times, render-only graph, C3, C5 window, NEXT-4 BA
for v in "$@"; do
  if [ "$v" = base ]; then unset CSPLAT_LIB; else export CSPLAT_LIB=variants/$v.so; fi
  timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sw_$v.json 2>gpurun_out/sw_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/sw_$v.json'));print('$v', round(d['value'],1), {k:round(v*1000,1) for k,v in d['stage_ms'].items()}, 'RO', round(d['render_only_graph']['ms_median']*1000,1), 'C3', round(d['tracking_c3']['ms_per_iter']*1000,1), 'C5', round(d['c5_window']['ms_per_window_iter'],2), 'BA', round(d['next_rows']['global_ba']['ms_per_iter'],3))"
done
unset CSPLAT_LIB
