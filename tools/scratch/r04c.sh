# ncu --set full of conv1 and conv3 (one full-batch launch each) for the shared-memory accounting
set -u
OUT=gpurun_out/r04c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv1_tc|k_conv3_r4" -s 2 -c 2 -o $OUT/prof13 python tools/time_stages.py lowrate 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof13.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null; wc -c $OUT/raw.csv
