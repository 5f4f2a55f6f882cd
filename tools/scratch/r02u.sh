python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_w3.so timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py -q -x -k "every_element or impulse or lowrate or invariants or multicast" 2>&1 | tail -2
bash tools/scratch/ab_lib.sh 3 product w3 2>&1
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_w3p.so timeout 300 python tools/time_stages.py lowrate 3 2>&1 | grep "conv2 cta" | head -3
