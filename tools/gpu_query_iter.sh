mkdir -p gpurun_out
timeout 300 python tools/bench_query.py > gpurun_out/bench_query.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "mlp or parity or quality" > gpurun_out/pytest_q.txt 2>&1
tail -3 gpurun_out/pytest_q.txt
