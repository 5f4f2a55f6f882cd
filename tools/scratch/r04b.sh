# bench with the training probe; A/B of a small first e2e chunk
set -u
OUT=gpurun_out/r04b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
timeout 600 python tools/scratch/ab_e2e_head.py > $OUT/ab_head.jsonl 2>&1; echo "ab rc=$?"
