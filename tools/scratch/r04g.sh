# conv2 zero-tap-slot skip v2 (copy issued first, zeros + arrival after): conv2/train tests, A/B, bench
set -u
OUT=gpurun_out/r04g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py tests/test_gpu_train.py tests/test_gpu_stack.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
bash tools/scratch/ab_lib_sustained.sh nozs > $OUT/ab.jsonl 2>&1
