# Round profile: launch list of one bench run, one ncu --set full capture of
# each hot kernel, summaries + traffic.json (GPU box).
#   bash tools/gpu_profile_round.sh <tag>
mkdir -p gpurun_out
TAG=${1:-r1}
# scene setup builds the BVHs on the GPU: keep those kernels out of the list
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  -k regex:"^(?!sah_|huge_|iota_kernel)" \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${TAG}_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gather_warp|query_ts" -c 3 -o gpurun_out/${TAG}_full -f \
  python bench.py --profile --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_full.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.md
python tools/ncu_summary.py full gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_summary.md
python tools/ncu_summary.py traffic gpurun_out/${TAG}_full.ncu-rep \
  "ncu --set full --clock-control none, profiles/${TAG}_ncu_full_summary.md (bench.py C2 workload, 1 launch each)" > gpurun_out/traffic.json
tail -3 gpurun_out/${TAG}_full.log
