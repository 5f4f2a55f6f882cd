# conv2 mixed row-block heights: targeted parity, then A/B against uniform 6-row blocks (alternating, same box)
set -u
OUT=gpurun_out/r02w; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
bash tools/scratch/ab_env.sh 3 "DI_EXP_C2_MIXED=1" "DI_EXP_C2_MIXED=0" > $OUT/ab.txt 2>&1; cat $OUT/ab.txt
timeout 600 python bench.py --no-cpu-configs > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cut -c1-600 $OUT/bench.json
