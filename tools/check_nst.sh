set -x
O=gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -3 > $O/n_pytest.txt
for v in "" _nst4 _nst8 _nst10 ""; do echo "== lib '$v'"; for c in 3d_512_l1 3d_512_l0; do GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200$v.so timeout 200 python tools/time_configs.py --only $c --reps 5; done; done > $O/n_configs.txt 2>&1
