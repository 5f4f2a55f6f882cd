# conv2 polling back-off: epilogue tfull waits / producer wempty waits with __nanosleep, A/B + ncu counts
set -u
OUT=gpurun_out/r04e; mkdir -p $OUT
bash tools/scratch/ab_lib_sustained.sh epi prod both > $OUT/ab.jsonl 2>&1
for L in libdeepinverse.so libdeepinverse_exp_epi.so libdeepinverse_exp_prod.so libdeepinverse_exp_both.so; do
  DI_LIB=paper_1701_03891_b200/$L timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:"k_conv2_tc" -s 2 -c 1 --csv python tools/time_stages.py lowrate 1 > $OUT/ncu_$L.csv 2>&1
done
