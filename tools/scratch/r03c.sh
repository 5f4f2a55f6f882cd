set -u
OUT=gpurun_out/r03c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python tools/scratch/wbw.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py tests/test_gpu_sensing.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for i in 1 2 3; do timeout 300 python tools/time_stages.py lowrate 20 2>&1 | tail -1 | cut -c1-200; done
