set -u
OUT=gpurun_out/r03b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/scratch/e2e_probe.py > $OUT/e2e.txt 2>&1; head -1 $OUT/e2e.txt
for i in 1 2 3; do timeout 300 python tools/time_stages.py lowrate 20 2>&1 | tail -1 | cut -c1-200; done
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 600 python bench.py --no-cpu-configs > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cut -c1-700 $OUT/bench.json
