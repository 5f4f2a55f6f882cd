python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_elementwise.py tests/test_gpu_parity.py tests/test_gpu_stack.py -q -x 2>&1 | tail -2
bash tools/scratch/ab_lib.sh 3 product ps4 2>&1
