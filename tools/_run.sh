for v in "" _tb2; do echo "== $v"; GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200$v.so python tools/time_configs.py --only 3d_512_l1; done > gpurun_out/tb2.txt 2>&1
GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200_tb2.so python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -5 >> gpurun_out/tb2.txt
