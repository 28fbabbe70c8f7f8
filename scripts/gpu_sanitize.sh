python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
