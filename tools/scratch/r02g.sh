OUT=gpurun_out/r02g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_sensing.py tests/test_gpu_train.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 $OUT/pytest.log
bash tools/scratch/ab_env.sh 2 "X=1" > $OUT/ab.txt 2>&1; cat $OUT/ab.txt
