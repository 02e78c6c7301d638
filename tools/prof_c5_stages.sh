# usage: bash tools/prof_c5_stages.sh (GPU box) -- C5 breakdown: per-stage times of three keyframes + the window's launch list
for kf in 0 21 42; do python tools/c5_stages.py $kf c5; done > gpurun_out/p3_stages.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3_c5_launches.csv python tools/prof_c5.py 1 > gpurun_out/p3_l.log 2>&1
cat gpurun_out/p3_stages.txt
