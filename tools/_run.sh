for v in _mb3 _mb4 _mb3ep2; do
  echo "== variant '$v'"
  GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200$v.so python tools/time_configs.py --only batch64_256
  GEODIST_LIB=paper_2208_00001_b200/lib/libgeodist_b200$v.so python tools/time_configs.py --only gsf
done > gpurun_out/mb.txt 2>&1
