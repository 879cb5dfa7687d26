# compute-sanitizer passes over the smoke path (small C1 scene: gather,
# labels, tcgen05 query, training step). Run on the GPU box.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool smoke exit $?"
  tail -2 gpurun_out/sanitize_$tool.txt
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python tools/sanitize_paths.py > gpurun_out/sanitize_paths_$tool.txt 2>&1
  echo "$tool paths exit $?"
  tail -2 gpurun_out/sanitize_paths_$tool.txt
done
