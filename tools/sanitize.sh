# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the step and tracking paths: bash tools/sanitize.sh (GPU box)
: > gpurun_out/r2i_sanitizers.txt
for t in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $t python tools/memcheck_step.py" >> gpurun_out/r2i_sanitizers.txt
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t python tools/memcheck_step.py 2>&1 | grep -v "^ok" | tail -4 >> gpurun_out/r2i_sanitizers.txt
done
cat gpurun_out/r2i_sanitizers.txt
