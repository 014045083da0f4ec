timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab2.txt
for v in "" _prev; do echo "== lib '$v'"; for c in 2d_512 3d_128 3d_512 gsf batch64_256; do GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200$v.so timeout 300 python tools/time_configs.py --only $c; done; done >> gpurun_out/ab2.txt 2>&1
