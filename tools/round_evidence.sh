#!/usr/bin/env bash
# Round-end evidence on one B200 (run from the repo root on the GPU box):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/round_evidence.sh r02'
# Writes gpurun_out/<tag>_*; the summaries worth keeping are copied into profiles/.
#   1. pytest -m gpu (parity, variants, the reference's own suites on the drop-in)
#   2. smoke(), bench.py (N = 1, 512^3), bench.py --impl reference, bench.py --config batch64
#   3. every BASELINE config timed (tools/time_configs.py) and checked at full size against
#      the reference (tools/parity_configs.py); the batch shards of N = 1/2/4/8 ranks
#   4. ncu: the launch list of one 512^3 transform, then --set full of one sweep launch of
#      the production clustered kernel (GEODIST_SWEEP_NOCOOP=1: ncu's kernel replay rejects
#      the cooperative + cluster launch; the grid is co-resident either way), each only
#      after the same command ran clean without ncu.
set -u
T=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_smi.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/${T}_pytest.txt 2>&1; tail -3 $O/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
timeout 900 python bench.py --config batch64 --steps 5 > $O/${T}_bench_batch.json 2> $O/${T}_bench_batch.err
timeout 900 python tools/time_configs.py --reps 5 > $O/${T}_configs.txt 2>&1
timeout 1800 python tools/parity_configs.py > $O/${T}_parity.jsonl 2> $O/${T}_parity.err
timeout 900 python tools/batch_shards.py > $O/${T}_batch_shards.txt 2>&1
GEODIST_SWEEP_NOCOOP=1 timeout 300 python tools/prof_step.py --reps 1 > $O/${T}_plain.log 2>&1 && \
GEODIST_SWEEP_NOCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${T}_launches.csv python tools/prof_step.py --reps 1 > $O/${T}_ncu_ll.log 2>&1
python tools/launch_list.py $O/${T}_launches.csv "one generalized_geodesic transform, 512^3, spacing (1,1,2.5), lambda=1, it=4" "python tools/prof_step.py --reps 1" > $O/${T}_launches_summary.csv 2>&1
GEODIST_SWEEP_NOCOOP=1 timeout 300 python tools/prof_step.py --reps 1 > $O/${T}_plain_nocoop.log 2>&1 && \
GEODIST_SWEEP_NOCOOP=1 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:sweep_kernel -c 1 -o $O/${T}_prof -f python tools/prof_step.py --reps 1 > $O/${T}_ncu_full.log 2>&1
python tools/ncu_summary.py $O/${T}_prof.ncu-rep 268435456 > $O/${T}_ncu_sweep.txt 2>&1
ncu -i $O/${T}_prof.ncu-rep --page raw --csv > $O/${T}_ncu_raw.csv 2>/dev/null
rm -f $O/${T}_prof.ncu-rep
