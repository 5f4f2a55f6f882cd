# shared-memory accesses as LDS / STS (aligned base by pointer arithmetic) vs generic LD / ST: A/B, ncu, tests
set -u
OUT=gpurun_out/r04j; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
bash tools/scratch/ab_lib_sustained.sh generic > $OUT/ab.jsonl 2>&1
for L in libdeepinverse.so libdeepinverse_exp_generic.so; do
  DI_LIB=paper_1701_03891_b200/$L timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum -k regex:"k_conv2_tc|k_conv1_tc|k_conv3_r4" -s 3 -c 3 --csv python tools/time_stages.py lowrate 1 > $OUT/ncu_$L.csv 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
