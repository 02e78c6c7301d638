# One GPU-box session: full bench, the 2-rank (gloo, one GPU) smoke of the
# multi-rank path, the reference arm, and the profile pass.
set -x
python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
CSPLAT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/r2d_mr.json 2> gpurun_out/r2d_mr.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2d_ref.json 2> gpurun_out/r2d_ref.err
bash tools/profile_round.sh r2 > /dev/null 2>&1
nproc; lscpu | grep "Model name"
