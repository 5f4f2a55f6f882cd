# conv2 mixed row-block heights + conv3 on image pairs (row-streamed): targeted parity, stage timing, A/B mixed
set -u
OUT=gpurun_out/r02w; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail $OUT/build.log; exit 1; }
timeout 300 python tools/time_stages.py lowrate 20 > $OUT/stages0.json 2>&1; cat $OUT/stages0.json | cut -c1-400
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py tests/test_gpu_sensing.py tests/test_gpu_stack.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -25 $OUT/pytest.log | cut -c1-300
bash tools/scratch/ab_env.sh 3 "DI_EXP_C2_MIXED=1" "DI_EXP_C2_MIXED=0" > $OUT/ab.txt 2>&1; cat $OUT/ab.txt
for c in larger stress tiny; do timeout 600 python tools/time_stages.py $c 20 >> $OUT/stages.jsonl 2>&1; done; cut -c1-300 $OUT/stages.jsonl
