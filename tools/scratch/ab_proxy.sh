for i in 1 2; do
for v in MB1 MB2; do
  if [ $v = MB1 ]; then export DI_EXP_PROXY_MB1=1; else unset DI_EXP_PROXY_MB1; fi
  for cfg in stress lowrate larger; do
    python tools/time_stages.py $cfg 10 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v','$cfg',d['stages_ms'][0],d['proxy_tflops'])"
  done
done; done
