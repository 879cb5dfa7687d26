# A/B of whole-library variants at C2 (gather alone + the whole pass):
#   bash tools/ab_libs.sh variants/libnif_a.so variants/libnif_b.so ...
# the in-tree build is always measured first as the baseline.
mkdir -p gpurun_out
for lib in paper_2306_07191_b200/libnif_b200.so "$@"; do
  echo "== $lib"
  NIF_B200_LIB=$lib timeout 300 python tools/ab_gather.py 0
done
