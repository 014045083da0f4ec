set -x
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > $O/f_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/f_smoke.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 > $O/f_bench.json 2> $O/f_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/f_bench_ref.json 2> $O/f_bench_ref.err
timeout 400 python tools/time_configs.py > $O/f_configs.txt 2>&1
