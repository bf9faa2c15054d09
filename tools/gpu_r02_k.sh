# round 2, call K: cross-batch pipelining (workspace slots, scan reserve) -- tests, N=1 probe, G=8 per-rank
# model, bench; workload reports of the latent-space generator
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_k.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_pipe_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pipe_k.log
timeout 900 python tools/overlap_probe.py --config C4 --reserve 0,4,8,12,16,24 > gpurun_out/overlap_c4_k.json 2> gpurun_out/overlap_c4_k.err
timeout 900 python tools/shard_model.py --config C4 --G 8 --batches 8 > gpurun_out/shard_model_c4_g8_k.json 2> gpurun_out/shard_model_c4_g8_k.err
timeout 1200 python bench.py > gpurun_out/bench_c4_k.json 2> gpurun_out/bench_c4_k.err
timeout 900 python tools/workload_report.py --config C2 > gpurun_out/workload_c2_k.json 2> gpurun_out/workload_c2_k.err
timeout 900 python tools/workload_report.py --config C3 > gpurun_out/workload_c3_k.json 2> gpurun_out/workload_c3_k.err
tail -3 gpurun_out/pytest_pipe_k.log; cat gpurun_out/overlap_c4_k.json; head -c 600 gpurun_out/bench_c4_k.json
# tcgen05 tensor-pipe evidence for K1: UTCHMMA fp16->fp32 op count vs 2*B*L*d
timeout 900 ncu --clock-control none --kernel-name regex:"k_filter_tc" --launch-skip 6 --launch-count 3 --csv \
  --metrics gpu__time_duration.sum,sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32.sum.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file gpurun_out/ncu_k1_tensor_k.csv python bench.py --steps 4 --warmup 3 --ncu --pipeline 0 > gpurun_out/ncu_k1_tensor_k.log 2>&1
timeout 600 python tools/scan_trace.py --config C4 --G 1 --release > gpurun_out/scan_trace_rel_k.jsonl 2> gpurun_out/scan_trace_rel_k.err
