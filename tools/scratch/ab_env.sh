# A/B of di_create-time switches on one box (lowrate, per-stage CUDA events): bash tools/scratch/ab_env.sh <rounds> "<VAR=val ...>" ...
R=$1; shift
for i in $(seq $R); do
  for v in "$@"; do
    env $v python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['stages_ms'],d['conv2_tflops'])"
  done
done
