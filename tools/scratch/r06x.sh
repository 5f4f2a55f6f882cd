# round-2 final evidence at HEAD (re-entry session): full GPU suite (product and DI_DEBUG library), bench twice, other
# configs, launch list, ncu --set full of the path kernels and of the stress lifting on CTA pairs, HBM floors, power, e2e
set -u
OUT=gpurun_out/r06x; mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1; nproc >> $OUT/gpu.txt; lscpu | grep 'Model name' >> $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
DI_NVCC_EXTRA=-DDI_DEBUG python paper_1701_03891_b200/build.py > $OUT/build_debug.log 2>&1 || echo DEBUG BUILD FAILED
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp.so timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_debug.log 2>&1; echo "debug pytest rc=$?"; tail -2 $OUT/pytest_debug.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err; echo "bench2 rc=$?"
for c in paper larger stress lowrate; do timeout 900 python tools/time_stages.py $c 20 >> $OUT/stages.jsonl 2>&1; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check --no-train --no-sustained"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_conv1_tc|k_conv2_tc|k_conv3_r4|k_proxy" -s 12 -c 4 -o $OUT/prof_all $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 1500 ncu --set full --clock-control none -k regex:"k_proxy_pair" -s 3 -c 1 -o $OUT/prof_pair python tools/time_stages.py stress 3 > $OUT/ncu_pair.log 2>&1; echo "ncu pair rc=$?"
ncu -i $OUT/prof_all.ncu-rep --page raw --csv > $OUT/raw_all.csv 2>/dev/null
./tools/scratch/hbm_probe > $OUT/hbm_probe.jsonl 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scratch/hbm_probe tools/scratch/hbm_probe.cu && ./tools/scratch/hbm_probe > $OUT/hbm_probe.jsonl 2>&1)
timeout 300 python tools/scratch/power_probe.py > $OUT/power.json 2>&1; tail -1 $OUT/power.json
timeout 300 python tools/scratch/e2e_probe.py > $OUT/e2e.txt 2>&1; head -1 $OUT/e2e.txt
