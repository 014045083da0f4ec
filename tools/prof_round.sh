# Round-end profiling: launch list, ncu --set full of the (clustered) sweep, and
# cluster-size experiments on every config.  Run on the GPU box from the repo root.
set -x
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python tools/prof_step.py --reps 1 > $O/ncu_ll.log 2>&1
python tools/launch_list.py $O/launches.csv "one generalized_geodesic transform, 512^3, spacing (1,1,2.5), lambda=1, it=4 (cluster-of-4 halo)" "python tools/prof_step.py --reps 1" > $O/launches_summary.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -c 1 \
  -o $O/prof_cluster -f python tools/prof_step.py --reps 1 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/prof_cluster.ncu-rep 268435456 > $O/ncu_sweep_cluster.txt 2>&1
rm -f $O/prof_cluster.ncu-rep
for cs in 0 2 4; do for c in 3d_512_l0 3d_512_l05 gsf_256 batch64_256x256x160 batch64_160x256x256 3d_128; do
  echo "== cs=$cs"; GEODIST_SWEEP_CLUSTER=$cs timeout 200 python tools/time_configs.py --only $c; done; done > $O/cluster_exp.txt 2>&1
