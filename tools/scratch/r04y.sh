# final: GPU suite at HEAD (product library), bench (sustained + training + thin layers), per-config stages, launch list
set -u
OUT=gpurun_out/r04y; mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1; nproc >> $OUT/gpu.txt; lscpu | grep 'Model name' >> $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err; echo "bench2 rc=$?"
for c in paper larger stress lowrate; do timeout 900 python tools/time_stages.py $c 20 >> $OUT/stages.jsonl 2>&1; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check --no-train --no-sustained"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
