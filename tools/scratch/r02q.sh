python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -q -x -k "lowrate or multicast or invariants or bf16 or sgd" 2>&1 | tail -2
bash tools/scratch/ab_env.sh 3 "DI_EXP_C2_WREP=1" "DI_EXP_C2_WREP=8" "DI_EXP_C2_WREP=32" 2>&1
