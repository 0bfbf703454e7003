# A/B of prebuilt libhxf.so variants (variants/*.so, swapped into _native/)
# on the bench workload; usage: bash tools/ab_variants.sh v1 v2 ...
cp paper_2109_04996_b200/_native/libhxf.so /tmp/libhxf.orig.so
for rep in 1 2; do
for v in "$@"; do
  cp variants/$v.so paper_2109_04996_b200/_native/libhxf.so
  timeout 300 python bench.py --steps 30 --no-cpu > gpurun_out/var_$v.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/var_$v.log') if l.startswith('{')][0]); print('$v', 'value', round(d['value'],2), 'k1_us', round(d['cg_iter']['operator_kernel_us'],2), 'apply_us', round(d['apply']['us'],2), 'frac', round(d['roofline']['frac'],3))"
done
done
cp /tmp/libhxf.orig.so paper_2109_04996_b200/_native/libhxf.so
