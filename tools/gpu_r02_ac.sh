# round 2, call AC: host-path query copies on a side stream (two staging buffers) -- tests, bench e2e
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_ac.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ac.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_ac.log
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 > gpurun_out/bench_ac.json 2> gpurun_out/bench_ac.err
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 --no-oracle --e2e-steps 40 > gpurun_out/bench_ac2.json 2> gpurun_out/bench_ac2.err
tail -2 gpurun_out/pytest_ac.log
for f in gpurun_out/bench_ac.json gpurun_out/bench_ac2.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['blocking_value']), d['e2e']['async_equal_to_blocking'])"; done
