#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/bench
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?"
python -c "
import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print(d['ms_per_step'], d['value'], r['frac']); print(json.dumps(r.get('random_access'), indent=1)); print(d['e2e'])"
tail -3 $O/bench.err
