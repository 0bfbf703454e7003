# A/B of prebuilt libhxf.so variants (variants/*.so) on timed single applies
# (tools/k1_time.py, K1ARGS selects the config); usage: bash tools/ab_k1_variants.sh v1 v2 ...
cp paper_2109_04996_b200/_native/libhxf.so /tmp/libhxf.orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp variants/$v.so paper_2109_04996_b200/_native/libhxf.so
    python tools/k1_time.py ${K1ARGS:-} --tag "$v"
  done
done
cp /tmp/libhxf.orig.so paper_2109_04996_b200/_native/libhxf.so
