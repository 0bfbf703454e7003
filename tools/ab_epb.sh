timeout 300 python tools/sweep.py --bp bp3 --p 7 --dims 31 > gpurun_out/epb_bp3.log 2>&1
timeout 300 python tools/sweep.py --bp bp5 --p 8 --sizes 1e7 > gpurun_out/epb_bp5.log 2>&1
timeout 300 python tools/sweep.py --bp bp2 --p 7 --sizes 1e7 > gpurun_out/epb_bp2.log 2>&1
timeout 300 python tools/sweep.py --bp bp4 --p 7 --sizes 1e7 > gpurun_out/epb_bp4.log 2>&1
timeout 300 python tools/sweep.py --bp bp1 --p 7 --sizes 1e7 > gpurun_out/epb_bp1.log 2>&1
