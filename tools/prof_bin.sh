# usage: bash tools/prof_bin.sh (GPU box) -- stand-alone C2 binning: launch list + full captures of the bucket pass and the sort
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_launches.csv python tools/bin_launches.py 3 > gpurun_out/p2_l.log 2>&1
for k in k_bucket k_sort_tiles; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/p2_$k python tools/bin_launches.py 2 > gpurun_out/p2_$k.log 2>&1
done
