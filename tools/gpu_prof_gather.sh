mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:gather_warp -c 1 -o gpurun_out/gather_full -f python tools/bench_gather.py > gpurun_out/ncu_gather.log 2>&1
tail -2 gpurun_out/ncu_gather.log
