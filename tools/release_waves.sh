# NEXT-4 experiment: release-mode scan vs wave count (C4, batch 256); one bench run per setting
export VLR_GEN_CACHE=/tmp/vlrcache
for z in 1 4 16; do
  VLR_RELEASE_WAVES=$z timeout 600 python bench.py --no-oracle --steps 20 > gpurun_out/rel_w$z.json 2> gpurun_out/rel_w$z.err
  python -c "import json; d=json.load(open('gpurun_out/rel_w$z.json')); print($z, json.dumps(d['release']))"
done
