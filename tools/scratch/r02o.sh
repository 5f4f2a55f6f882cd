python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py -q -x -k "every_element or impulse or lowrate or larger or multicast or ragged" 2>&1 | tail -3
bash tools/scratch/ab_env.sh 3 "X=1" "DI_EXP_C2_SPLIT=253" 2>&1
