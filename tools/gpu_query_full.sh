mkdir -p gpurun_out
V=${1:-1}
K=${2:-"tc2_kernel<\\(int\\)5, \\(int\\)3, \\(int\\)48, \\(int\\)3, \\(int\\)2, \\(int\\)6"}
timeout 600 ncu --set full --import-source on --kernel-name-base demangled -k "regex:$K" -c 1 -o gpurun_out/query2_full -f python tools/bench_query.py $V 1 > gpurun_out/ncu_query2.log 2>&1
tail -2 gpurun_out/ncu_query2.log
