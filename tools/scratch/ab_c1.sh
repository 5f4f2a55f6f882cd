for i in 1 2; do
for v in base DI_EXP_C1_L2ONLY; do
  if [ $v = base ]; then X=""; else X="-D$v"; fi
  DI_NVCC_EXTRA="$X" python paper_1701_03891_b200/build.py --force > /dev/null 2>&1
  python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['stages_ms'])"
done; done
