timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gt_ring.log 2>&1; tail -3 gpurun_out/gt_ring.log
timeout 600 bash tools/sweep_bwd.sh new
export CSPLAT_SINGLE_STREAM=1
ncu --set full --import-source on --clock-control none -k regex:"k_render_bwd" -s 1 -c 1 -o gpurun_out/ringP python tools/prof_step.py 2 > gpurun_out/ringP.log 2>&1
ncu -i gpurun_out/ringP.ncu-rep --page source --csv --print-source sass > gpurun_out/ringP_sass.csv 2>&1
