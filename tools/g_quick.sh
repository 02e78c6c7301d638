# quick GPU check: GPU tests + bench stage times (no oracle baseline)
TAG=${1:-q}
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/${TAG}_tests.log
python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_tests.log
python -c "
import json;d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('value',round(d['value']),'stage',{k:round(v*1000,1) for k,v in d['stage_ms'].items()},'ro',round(d['render_only_graph']['renders_per_s']),'c5',round(d['c5_window']['ms_per_window_iter'],2),'c3',round(d['tracking_c3']['ms_per_iter'],4),'ba',round(d['next_rows']['global_ba']['ms_per_iter'],3),'clk',d['clocks'])"
