set -x
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $O/rc2_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 3 > $O/rc2_bench.json 2> $O/rc2_bench.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:row_chain -c 1 \
  -o $O/prof_rc -f python tools/prof_step.py --reps 1 --shape 512,512 --spacing 1,1 --iters 2 > $O/ncu_rc.log 2>&1
ncu -i $O/prof_rc.ncu-rep --page raw --csv > $O/prof_rc_raw.csv 2>&1
ncu -i $O/prof_rc.ncu-rep --page details > $O/prof_rc_details.txt 2>&1
