mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_query_variants.py tests/test_gpu_mlp.py -x -q > gpurun_out/pytest_q.txt 2>&1
tail -2 gpurun_out/pytest_q.txt
timeout 1500 python tools/sweep_c5.py --out gpurun_out/c5_sweep.json > gpurun_out/c5_sweep.txt 2>&1
tail -1 gpurun_out/c5_sweep.txt
