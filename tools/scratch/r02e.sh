OUT=gpurun_out/r02e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "proxy_on_cta_pairs" > $OUT/pytest_pair_debug.log 2>&1; echo "pair debug rc=$?"; tail -15 $OUT/pytest_pair_debug.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "proxy_on_cta_pairs" > $OUT/pytest_pair.log 2>&1; echo "pair rc=$?"; tail -3 $OUT/pytest_pair.log
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_p3.so timeout 300 python tools/time_stages.py lowrate 5 > $OUT/prof3.txt 2>&1; grep conv3 $OUT/prof3.txt | tail -8
for v in X=1 DI_EXP_PROXY_PAIR=1 X=1 DI_EXP_PROXY_PAIR=1; do env $v timeout 600 python tools/time_stages.py larger 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('larger $v',d['stages_ms'])"; done
for v in X=1 DI_EXP_PROXY_PAIR=1 X=1 DI_EXP_PROXY_PAIR=1; do env $v timeout 900 python tools/time_stages.py stress 10 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('stress $v',d['stages_ms'])"; done
