for v in "HXF_DMMA_NW=4" "HXF_DMMA_NW=8" "HXF_PDL=1" "HXF_DMMA_NW=2"; do
  env $v timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/abk1_$v.log 2>&1
done
