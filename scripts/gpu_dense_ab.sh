python -c "import __graft_entry__ as g; g.build()" > /dev/null
echo "== plain"; python scripts/dense_perf.py 16384; python scripts/dense_perf.py 16384
cp paper_1707_01007_b200/csrc/dense.cu /tmp/dense_plain.cu
cp scripts/dense_variant_sleepy.cu paper_1707_01007_b200/csrc/dense.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null
echo "== sleepy"; python scripts/dense_perf.py 16384; python scripts/dense_perf.py 16384
cp /tmp/dense_plain.cu paper_1707_01007_b200/csrc/dense.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null
echo "== plain again"; python scripts/dense_perf.py 16384
