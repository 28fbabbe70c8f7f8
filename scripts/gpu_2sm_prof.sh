set -x
python -c "import __graft_entry__ as g; g.build()"
CFPQ_DENSE_2SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense2sm -s 3 -c 1 -o gpurun_out/prof_2sm python scripts/dense_perf.py 16384 2 > gpurun_out/ncu_2sm.txt 2>&1
tail -3 gpurun_out/ncu_2sm.txt
