timeout 1700 python tools/sweep.py --bp bp5 --p 2,3,5,7,10,15 --sizes 1e8 --out gpurun_out/sweep_bp5_1e8.md --csv gpurun_out/sweep_bp5_1e8.csv > gpurun_out/sweep_bp5_1e8.log 2>&1
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
