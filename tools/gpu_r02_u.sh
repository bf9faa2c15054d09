# round 2, call U: the other configurations / variants on the final build (bench lines)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_u.log 2>&1
timeout 900 python bench.py --config C2 --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c2_u.json 2> gpurun_out/bench_c2_u.err
timeout 900 python bench.py --config C3 --hot-mass 0.5 --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c3_h05_u.json 2> gpurun_out/bench_c3_h05_u.err
timeout 1200 python bench.py --config C4 --nbits 4 --m 256 --lat-batches 0 --sustained-s 0 --no-oracle > gpurun_out/bench_c4_pq4_u.json 2> gpurun_out/bench_c4_pq4_u.err
timeout 900 python bench.py --config C2 --metric 1 --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c2_ip_u.json 2> gpurun_out/bench_c2_ip_u.err
timeout 900 python bench.py --config C4 --nprobe 2048 --k 25 --steps 10 --lat-batches 0 --sustained-s 0 --no-oracle > gpurun_out/bench_c4_np2048_k25_u.json 2> gpurun_out/bench_c4_np2048_k25_u.err
for f in gpurun_out/bench_*_u.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['roofline']['frac'], (d.get('parity_sample') or {}).get('pass'))"; done
