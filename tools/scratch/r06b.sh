# conv1 phase-stacked form: parity (element-wise + path) and stage times
set -u
OUT=gpurun_out/r06b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_elementwise.py -m gpu -x -q > $OUT/pytest_elem.log 2>&1; echo "elem rc=$?"; tail -15 $OUT/pytest_elem.log
timeout 300 python tools/time_stages.py lowrate 20 > $OUT/stages.jsonl 2>&1; echo "stages rc=$?"; tail -3 $OUT/stages.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -5 $OUT/pytest_parity.log
