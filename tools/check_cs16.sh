O=gpurun_out
for env in "GEODIST_SWEEP_CLUSTER=0" "GEODIST_SWEEP_CLUSTER=8" "GEODIST_SWEEP_CLUSTER=16"; do
  echo "== $env"; for c in 3d_128 gsf_256 probe_256x256x160 probe_256x256x256; do env $env timeout 200 python tools/time_configs.py --only $c --reps 5; done; done > $O/cs16_configs.txt 2>&1
