# round 2, call Q: NEXT-4 with the alternating segment order + release-rest kernel, at 1/2/4 waves (C4)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_q.log 2>&1
for z in 1 2 4; do
  VLR_RELEASE_WAVES=$z timeout 900 python bench.py --no-oracle --steps 20 --lat-batches 0 --sustained-s 0 --e2e-steps 4 \
    > gpurun_out/rel_q_w$z.json 2> gpurun_out/rel_q_w$z.err
  python -c "import json; d=json.loads(open('gpurun_out/rel_q_w$z.json').read().strip().splitlines()[-1]); print($z, json.dumps(d['release']))"
done
