set -u
OUT=gpurun_out/r03a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/scratch/e2e_probe.py > $OUT/e2e.txt 2>&1; head -3 $OUT/e2e.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for i in 1 2 3; do timeout 300 python tools/time_stages.py lowrate 20 2>&1 | tail -1 | cut -c1-200; done
