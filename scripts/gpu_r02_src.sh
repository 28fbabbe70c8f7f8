#!/bin/bash
# Source-level ncu capture of closure_kernel (config 4) + TLB probe numbers.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/src
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 5 -c 1 \
   -o $O/prof_c4 python bench.py --workload config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > $O/ncu.txt 2>&1
ncu -i $O/prof_c4.ncu-rep --page source --csv --print-source sass > $O/src_sass.csv 2>&1
ncu -i $O/prof_c4.ncu-rep --page source --csv --print-source cuda > $O/src_cuda.csv 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tlb scripts/tlb_probe.cu && timeout 300 /tmp/tlb > $O/tlb.txt 2>&1
python scripts/phase_profile.py config4 > $O/phase.txt 2>&1
ls -la $O; cat $O/tlb.txt
