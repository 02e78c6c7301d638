# A/B library variants built by tools/variants.py (names as arguments): C2 step,
# stage times, C5 window and the NEXT-4 BA iteration
for v in "$@"; do
  CSPLAT_LIB=variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sw_$v.json 2>gpurun_out/sw_$v.err
  python -c "
import json,sys;d=json.load(open('gpurun_out/sw_$v.json'));print('$v', round(d['value'],1), {k:round(v*1000,1) for k,v in d['stage_ms'].items()}, 'C5', round(d['c5_window']['ms_per_window_iter'],2), 'BA', round(d['next_rows']['global_ba']['ms_per_iter'],3), 'render_only', round(d['render_only_graph']['ms_median']*1000,1))"
done
