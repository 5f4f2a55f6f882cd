python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
bash tools/scratch/ab_lib.sh 3 product r7 2>&1
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_p2.so timeout 300 python tools/time_stages.py lowrate 3 2>&1 | grep "conv2 cta" | head -4
