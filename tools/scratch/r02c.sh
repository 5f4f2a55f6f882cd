set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
bash tools/scratch/ab_lib.sh 2 product pf0 pf3 pf12 > $OUT/ab_pf.txt 2>&1; cat $OUT/ab_pf.txt
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-oracle-check"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_conv1_tc|k_conv3_r4" -s 2 -c 2 -o $OUT/prof_c13 $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 $OUT/ncu_full.log
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp.so timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_debug.log 2>&1; echo "debug pytest rc=$?"; tail -3 $OUT/pytest_debug.log
