timeout 200 python tools/time_configs.py --only 3d_512 > gpurun_out/bc.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/bc.txt
