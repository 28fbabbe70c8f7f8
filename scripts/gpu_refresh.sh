# refresh the round's bench lines and ncu evidence (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/nvsmi.txt
for W in config4 configS config3 config5 config2; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 600 python bench.py --workload configS --tensor-format 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_configS_int8.json 2> gpurun_out/bench_configS_int8.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1
# launch lists (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config4.csv \
   python bench.py --workload config4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_configS.csv \
   python bench.py --workload configS --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_rows_config4.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > /dev/null 2>&1
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:closure_kernel -s 5 -c 1 \
   -o gpurun_out/prof_config4 python bench.py --workload config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-supplementary > gpurun_out/ncu_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense2sm_kernel -s 20 -c 1 \
   -o gpurun_out/prof_configS python bench.py --workload configS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cS.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_scatter_kernel -s 6 -c 1 -o gpurun_out/prof_rows_scatter \
   python -c "
import sys; sys.path.insert(0,'.')
import torch, inputs as I
from paper_1707_01007_b200 import cfpq as C
w=I.config4_workload(); g=C.Grammar.from_workload(w); d=C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
r=C.closure(g,d,path_policy=3)
" > gpurun_out/ncu_rows.txt 2>&1
tail -2 gpurun_out/ncu_c4.txt gpurun_out/ncu_cS.txt gpurun_out/ncu_rows.txt
python scripts/phase_profile.py config4 > gpurun_out/phase_config4.txt 2>&1
python scripts/e2e_breakdown.py > gpurun_out/e2e_config4.txt 2>&1
ls -la gpurun_out | head -50
