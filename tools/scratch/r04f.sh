# conv2 zero-tap-slot skip: GPU suite, then A/B against the copy-everything build (burst + sustained), bench
set -u
OUT=gpurun_out/r04f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
bash tools/scratch/ab_lib_sustained.sh nozs > $OUT/ab.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
