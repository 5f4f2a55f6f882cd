python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_train.py -q -x 2>&1 | tail -2
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_r7.so timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py -q -x -k "every_element or impulse or lowrate or larger or invariants or shard or multicast" 2>&1 | tail -2
DI_DEBUG_MC=1 DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_r7.so python tools/time_stages.py lowrate 3 2>&1 | grep -i "conv2:" | head -2
bash tools/scratch/ab_lib.sh 3 product r7 2>&1
