OUT=gpurun_out/r02f; mkdir -p $OUT
SKIP_NCU=1 bash tools/gpu_check.sh r02f
python tools/time_stages.py lowrate 20 > $OUT/stages.json 2>&1; cat $OUT/stages.json
