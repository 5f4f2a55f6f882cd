# round-2 final check at the last commit: build from clean, GPU suite, smoke(), default bench, reference arm
set -u
OUT=gpurun_out/r06z; mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1; nproc >> $OUT/gpu.txt; lscpu | grep 'Model name' >> $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err; echo "bench2 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
head -c 1500 $OUT/bench2.json
