# conv2 weight copies split over two producer threads: tests, A/B against one producer, issuer profile
set -u
OUT=gpurun_out/r04i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py tests/test_gpu_train.py tests/test_gpu_stack.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
bash tools/scratch/ab_lib_sustained.sh oneprod > $OUT/ab.jsonl 2>&1
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_prof.so python tools/time_stages.py lowrate 1 2>&1 | grep "conv2 cta 0:\|stages" | cut -c1-330 > $OUT/prof.txt
