# round 2, call M: K1 query tile >= 1 CTA/SM, K3b rank select, K2 warp-aggregated histograms, release-merger
# experiment, G=8 launch list, sanitizers on the new paths, tests, C4 sweep + C3 residency grid
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_m.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.log
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_m.json 2> gpurun_out/shard_model_c4_g8_m.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^(k_|void k_)" \
  --launch-skip 400 --launch-count 300 --csv --log-file gpurun_out/launches_shard_g8_m.csv \
  python tools/shard_model.py --config C4 --G 8 --batches 4 --pipe-reserve "" > gpurun_out/ncu_shard_m.log 2>&1
VLR_REL_EXPERIMENT=1 timeout 600 python tools/scan_trace.py --config C4 --G 1 --release --release-nowait > gpurun_out/scan_trace_relexp_m.jsonl 2> gpurun_out/scan_trace_relexp_m.err
VLR_REL_EXPERIMENT=1 VLR_RELEASE_WAVES=1 timeout 600 python tools/scan_trace.py --config C4 --G 1 --release --release-nowait > gpurun_out/scan_trace_relexp_z1_m.jsonl 2> gpurun_out/scan_trace_relexp_z1_m.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_${tool}_m.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_m.log
done
timeout 1200 python bench.py > gpurun_out/bench_c4_m.json 2> gpurun_out/bench_c4_m.err
timeout 1500 python bench.py --lat-batches 0 --sustained-s 0 --no-oracle --steps 10 --sweep-out gpurun_out/sweep_c4_m.jsonl > gpurun_out/bench_c4_sweep_m.json 2> gpurun_out/bench_c4_sweep_m.err
bash tools/c3_grid.sh
tail -3 gpurun_out/pytest_m.log
