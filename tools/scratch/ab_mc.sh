timeout 300 python tools/time_stages.py lowrate 5 > /dev/null 2>&1; echo "warm rc=$?"
for i in 1 2 3; do
for v in MC NOMC; do
  if [ $v = NOMC ]; then export DI_EXP_NO_MC=1; else unset DI_EXP_NO_MC; fi
  timeout 300 python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['stages_ms'],d['conv2_tflops'])"
done; done
