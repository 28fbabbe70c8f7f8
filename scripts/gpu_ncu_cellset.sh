python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -c 2 -o gpurun_out/cellset -f python scripts/cellset_pair.py > gpurun_out/ncu_cellset.txt 2>&1
tail -5 gpurun_out/ncu_cellset.txt
