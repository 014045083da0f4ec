O=gpurun_out
for env in "" "GEODIST_SWEEP_R=2" "GEODIST_SWEEP_R=2 GEODIST_SWEEP_CLUSTER=2" "GEODIST_SWEEP_R=2 GEODIST_SWEEP_CLUSTER=4" "GEODIST_SWEEP_R=8"; do
  echo "== $env"; for c in 3d_128 gsf_256; do env $env timeout 200 python tools/time_configs.py --only $c --reps 5; done; done > $O/r2_configs.txt 2>&1
