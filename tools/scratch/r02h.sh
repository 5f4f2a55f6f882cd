OUT=gpurun_out/r02h; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_sensing.py tests/test_gpu_train.py -q -x 2>&1 | tail -15
