# C3 residency grid: alpha x hot mass, one bench line each (gen3 workload: latent-space
# generator with k-means lists). Latency / sustained / oracle legs off to bound the run.
export VLR_GEN_CACHE=/tmp/vlrcache
out=gpurun_out/c3_grid.jsonl
: > $out
for al in 0.8 1.0 1.4; do
  for hm in 0.3 0.5 0.7; do
    timeout 900 python bench.py --config C3 --alpha $al --hot-mass $hm --steps 20 --warmup 3 --no-oracle \
      --lat-batches 0 --sustained-s 0 >> $out 2>> gpurun_out/c3_grid.err || echo "{\"failed\": \"alpha $al hot $hm\"}" >> $out
  done
done
