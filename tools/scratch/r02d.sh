OUT=gpurun_out/r02d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py -x -q -k "impulse or every_element or multicast or lowrate or larger" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
bash tools/scratch/ab_env.sh 3 "X=1" "DI_EXP_C2_CLUSTER=4" "DI_EXP_NO_MC=1" > $OUT/ab.txt 2>&1; cat $OUT/ab.txt
