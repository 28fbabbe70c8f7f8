#!/bin/bash
# round-2 evidence: bench lines of every workload + reference arm, launch lists, ncu full
# captures of the dominant kernels (run under gpurun; summaries are made here afterwards)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/nvsmi.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_config4.json 2> $O/bench_config4.err
for W in configS config3 config5 config2; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > $O/bench_$W.json 2> $O/bench_$W.err
done
timeout 600 python bench.py --workload config3 --schedule 3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config3_gs.json 2>&1
timeout 600 python bench.py --workload config4 --schedule 3 --steps 10 --warmup 3 --no-cpu-baseline --no-supplementary > $O/bench_config4_gs.json 2>&1
timeout 600 python bench.py --workload configS --tensor-format 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_configS_int8.json 2> $O/bench_configS_int8.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>&1
timeout 600 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --force-sharded --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun1_sharded.json 2> $O/bench_torchrun1_sharded.err
# launch lists (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config4.csv \
   python bench.py --workload config4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_configS.csv \
   python bench.py --workload configS --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches_rows_config4.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > /dev/null 2>&1
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 5 -c 1 \
   -o $O/prof_config4 python bench.py --workload config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > $O/ncu_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense2sm_kernel -s 20 -c 1 \
   -o $O/prof_configS python bench.py --workload configS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_cS.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_scatter_kernel -s 6 -c 1 -o $O/prof_rows_scatter \
   python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > $O/ncu_rows_scatter.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_rpush_kernel -s 6 -c 1 -o $O/prof_rows_rpush \
   python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > $O/ncu_rows.txt 2>&1
python scripts/phase_profile.py config4 > $O/phase_config4.txt 2>&1
python scripts/c4_variants.py > $O/c4_variants.txt 2>&1
python scripts/e2e_breakdown.py > $O/e2e_config4.txt 2>&1
ls -la $O
