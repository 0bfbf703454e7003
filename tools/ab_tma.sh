# A/B of the TMA slab gather in the DMMA kernel (HXF_TMA=0: per-lane loads)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_surface.py tests/test_gpu_api.py -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
for v in 1 0 1 0; do HXF_TMA=$v timeout 300 python bench.py --steps 30 --no-cpu > gpurun_out/tma_$v.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/tma_$v.log') if l.startswith('{')][0]); print('TMA=$v', 'value', round(d['value'],2), 'k1_us', round(d['cg_iter']['operator_kernel_us'],2), 'apply_us', round(d['apply']['us'],2), 'frac', round(d['roofline']['frac'],3))"; done
for v in 1 0; do HXF_TMA=$v timeout 300 python tools/sweep.py --bp bp6 --p 6,7 --sizes 4.1e7 --out gpurun_out/tma_bp6_$v.md > /dev/null 2>&1; echo "TMA=$v"; cat gpurun_out/tma_bp6_$v.md | tail -3; done
