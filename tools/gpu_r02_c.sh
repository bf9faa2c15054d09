# round 2, call C: new generator (k-means lists, hierarchical topics) through the GPU tests, workload
# reports, ncu evidence for K1 (single vs pair), K2, K3a, the tcgen05 metric list, the G=8 launch list
set -x
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_c.log 2>&1
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt; lscpu | grep -i "model name" >> gpurun_out/host_mem.txt
timeout 120 ncu --query-metrics > gpurun_out/ncu_query_metrics.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02_c.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r02_c.log
timeout 900 python tools/workload_report.py --config C2 > gpurun_out/workload_c2.json 2> gpurun_out/workload_c2.err
timeout 600 env K1_VARIANT=single VLR_FILTER_PAIR=0 ncu --set full --import-source on --clock-control none -k regex:"k_filter|k_select|k_exact|k_qprep" -s 12 -c 8 -o gpurun_out/prof_k1_single -f python tools/k1_bench.py --child --config C4 --iters 2 > gpurun_out/ncu_k1_single.log 2>&1
timeout 600 env K1_VARIANT=pair VLR_FILTER_PAIR=1 ncu --set full --import-source on --clock-control none -k regex:"k_filter_pair" -s 3 -c 2 -o gpurun_out/prof_k1_pair -f python tools/k1_bench.py --child --config C4 --iters 2 > gpurun_out/ncu_k1_pair.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shard_g8.csv python tools/shard_model.py --config C3 --G 8 --batches 2 --warmup 1 > gpurun_out/ncu_shard.log 2>&1
timeout 900 python tools/workload_report.py --config C3 > gpurun_out/workload_c3.json 2> gpurun_out/workload_c3.err
tail -3 gpurun_out/pytest_gpu_r02_c.log
