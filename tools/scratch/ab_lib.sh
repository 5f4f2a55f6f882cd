# A/B of experiment libraries on one box (lowrate bench workload, per-stage CUDA events):
#   bash tools/scratch/ab_lib.sh <rounds> <lib>...   (lib "product" = libdeepinverse.so)
R=$1; shift
for i in $(seq $R); do
  for v in "$@"; do
    if [ "$v" = product ]; then unset DI_LIB; else export DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_$v.so; fi
    python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['stages_ms'],d['conv2_tflops'])"
  done
done
unset DI_LIB
