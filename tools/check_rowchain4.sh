set -x
O=gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_variants_gpu.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -5 > $O/rc4_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/rc4_smoke.txt 2>&1
for rc in 1 0; do echo "== GEODIST_ROWCHAIN=$rc"; GEODIST_ROWCHAIN=$rc timeout 200 python tools/time_configs.py --only 2d_512 --reps 5; done > $O/rc4_configs.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:row_chain -c 1 \
  -o $O/prof_rc4 -f python tools/prof_step.py --reps 1 --shape 512,512 --spacing 1,1 --iters 2 > $O/ncu_rc4.log 2>&1
