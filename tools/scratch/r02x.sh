set -u
OUT=gpurun_out/r02x; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
DI_NVCC_EXTRA="-DDI_PROF_CONV3" DI_EXP_NAME=prof3 python paper_1701_03891_b200/build.py > $OUT/build_prof.log 2>&1 || echo PROF BUILD FAILED
timeout 300 python tools/scratch/diag_w.py 64 4096 0,1,51,4095 2>&1 | tail -4
timeout 300 python tools/scratch/diag_w.py 64 7 0,5,6 2>&1 | tail -3
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_prof3.so timeout 300 python tools/time_stages.py lowrate 3 2>&1 | tail -5
for i in 1 2; do timeout 300 python tools/time_stages.py lowrate 20 2>&1 | tail -1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py tests/test_gpu_sensing.py tests/test_gpu_stack.py tests/test_gpu_train.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest.log | cut -c1-300
