# Row-chain (2D) kernel + spatial cluster default: parity, timings, ncu (L2-only sweep variant:
# the clustered cooperative sweep traps under ncu replay).
set -x
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $O/rc_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/rc_smoke.txt 2>&1
for rc in 1 0; do echo "== GEODIST_ROWCHAIN=$rc"; GEODIST_ROWCHAIN=$rc timeout 200 python tools/time_configs.py --only 2d_512; done > $O/rc_configs.txt 2>&1
timeout 200 python tools/time_configs.py --only 3d_512_l0 >> $O/rc_configs.txt 2>&1
GEODIST_SWEEP_CLUSTER=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches0.csv python tools/prof_step.py --reps 1 > $O/ncu_ll0.log 2>&1
python tools/launch_list.py $O/launches0.csv "one generalized_geodesic transform, 512^3, spacing (1,1,2.5), lambda=1, it=4 (GEODIST_SWEEP_CLUSTER=0: L2-only halo links)" "GEODIST_SWEEP_CLUSTER=0 python tools/prof_step.py --reps 1" > $O/launches0_summary.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches2d.csv python tools/prof_step.py --reps 1 --shape 512,512 --spacing 1,1 --iters 2 > $O/ncu_ll2d.log 2>&1
python tools/launch_list.py $O/launches2d.csv "2D 512x512 lambda=1 it=2 (row-chain kernel)" "python tools/prof_step.py --reps 1 --shape 512,512 --spacing 1,1 --iters 2" > $O/launches2d_summary.csv
