# mbarrier try_wait suspend-time hints: bench-style burst + sustained A/B, and ncu of conv2 with the 100-us hint
set -u
OUT=gpurun_out/r04d; mkdir -p $OUT
bash tools/scratch/ab_lib_sustained.sh h1000 h100000 h10000000 > $OUT/ab.jsonl 2>&1
for L in libdeepinverse.so libdeepinverse_exp_h100000.so; do
  DI_LIB=paper_1701_03891_b200/$L timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed_op_shared_ld.sum -k regex:"k_conv2_tc|k_conv1_tc|k_conv3_r4" -s 6 -c 3 --csv python tools/time_stages.py lowrate 1 > $OUT/ncu_$L.csv 2>&1
done
