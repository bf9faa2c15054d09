# round 2, call AB: PDL off under stream capture -- latency (CUDA graph) leg + sustained, release tests
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "graph or capture or reserve or c1" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
timeout 1200 python bench.py --no-oracle --steps 20 --e2e-steps 4 > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
VLR_PDL=0 timeout 1200 python bench.py --no-oracle --steps 20 --e2e-steps 4 > gpurun_out/bench_ab_nopdl.json 2> gpurun_out/bench_ab_nopdl.err
for f in gpurun_out/bench_ab.json gpurun_out/bench_ab_nopdl.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), {b: round(v['p50_ms'],3) for b,v in d['latency']['by_batch'].items()}, round(d['latency']['sustained']['qps_all']))"; done
