set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r01b.json 2> gpurun_out/ref_r01b.err
python tools/prof_step.py --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python tools/prof_step.py --reps 1 > gpurun_out/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -c 1 -o gpurun_out/prof_r01b_sweep -f python tools/prof_step.py --reps 1 > gpurun_out/ncu_s.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:transpose -c 1 -o gpurun_out/prof_r01b_transpose -f python tools/prof_step.py --reps 1 > gpurun_out/ncu_t.log 2>&1
tail -2 gpurun_out/ncu_s.log
