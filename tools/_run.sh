timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for rw in -1 0; do echo "== RW=$rw"; GEODIST_SWEEP_RW=$rw timeout 120 python tools/time_configs.py --only 3d_512; done > gpurun_out/rw2.txt 2>&1
