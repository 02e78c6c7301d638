# One GPU-box session for the round's evidence: bench, reference arm, the
# 2-rank gloo smoke of the multi-rank path, smoke(), profiles (compute-sanitizer
# is closed on the GPU pool since round 2's session 3).
# usage: bash tools/box_final.sh <tag>
TAG=${1:-r2i}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_ref.err
CSPLAT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_multirank_gloo.json 2> gpurun_out/${TAG}_mr.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
bash tools/profile_round.sh $TAG > /dev/null 2>&1
ls gpurun_out | grep $TAG
