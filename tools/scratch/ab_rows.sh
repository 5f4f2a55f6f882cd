# A/B of the conv2 unit height on one box: R=6 vs R=7 (lowrate bench workload, CUDA events).
# Geometry overrides build the EXPERIMENT library (build.py: libdeepinverse_exp.so); DI_LIB points the binding at it.
export DI_LIB=paper_1701_03891_b200/libdeepinverse_exp.so
for i in 1 2; do
for r in 6 7; do
  DI_NVCC_EXTRA=-DDI_C2_ROWS=$r python paper_1701_03891_b200/build.py --force > /dev/null 2>&1
  DI_NVCC_EXTRA=-DDI_C2_ROWS=$r python tools/time_stages.py lowrate 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('R$r',d['stages_ms'],d['conv2_tflops'])"
done; done
