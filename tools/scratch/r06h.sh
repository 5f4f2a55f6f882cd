# conv2: L2 prefetch of the next unit's strip one unit ahead (experiment library) against the product, alternating
set -u
OUT=gpurun_out/r06h; mkdir -p $OUT
for i in 1 2 3; do
  timeout 300 python tools/time_stages.py lowrate 20 >> $OUT/stages_product.jsonl 2>&1
  DI_LIB=paper_1701_03891_b200/libdeepinverse_exp.so timeout 300 python tools/time_stages.py lowrate 20 >> $OUT/stages_pf.jsonl 2>&1
done
echo product; grep -h stages_ms $OUT/stages_product.jsonl | cut -c1-140; echo prefetch; grep -h stages_ms $OUT/stages_pf.jsonl | cut -c1-140
