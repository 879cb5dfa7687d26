mkdir -p gpurun_out
./tools/mma_lat > gpurun_out/mma_lat.txt 2>&1
timeout 300 python tools/probe_query.py > gpurun_out/probe_query.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:query_tc_kernel -c 2 -o gpurun_out/query_full -f python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_query.log 2>&1
tail -3 gpurun_out/ncu_query.log
