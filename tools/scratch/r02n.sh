python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_p3.so timeout 300 python tools/time_stages.py lowrate 3 2>&1 | grep "conv3 cta" | head -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv3_r4 -s 3 -c 1 -o gpurun_out/r02n_c3 python tools/time_stages.py lowrate 3 > /dev/null 2>&1; echo "ncu rc=$?"
