# round 2, call Y: release scan without the wave-loop registers (spills 28 -> 16 B, none in the hot loop):
# release vs plain device time (events) with the product library, release tests, bench release leg
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_y.log 2>&1
timeout 900 python -m pytest tests/test_gpu_release.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/pytest_y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.log
timeout 900 python tools/release_probe.py 128000000 1024 65536 128 128 256 > gpurun_out/release_probe_c4_y.json 2> gpurun_out/release_probe_c4_y.err
timeout 900 python tools/release_timeline.py --config C4 > gpurun_out/release_timeline_y.json 2> gpurun_out/release_timeline_y.err
timeout 900 python bench.py --no-oracle --steps 20 --lat-batches 0 --sustained-s 0 --e2e-steps 4 > gpurun_out/bench_rel_y.json 2> gpurun_out/bench_rel_y.err
tail -2 gpurun_out/pytest_y.log; cat gpurun_out/release_probe_c4_y.json
