for i in 1 2; do
for v in base DI_EXP_NOEPI_SMEM DI_EXP_HALFW; do
  if [ $v = base ]; then X=""; else X="-D$v"; fi
  DI_NVCC_EXTRA="$X" python paper_1701_03891_b200/build.py --force > /dev/null 2>&1
  python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v',d['stages_ms'],d['conv2_tflops'])"
done; done
