#!/bin/bash
# One gpurun call: build, GPU tests, bench, ncu launch list + one --set full capture of conv layer 2.
# usage (from repo root, on the GPU box): bash tools/gpu_check.sh [tag] [pytest-args...]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt 2>&1; nproc >> $OUT/gpu.txt; lscpu | grep 'Model name' >> $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m "${PYTEST_MARK:-gpu}" -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err
if [ "${SKIP_NCU:-0}" != 1 ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  $CMD > $OUT/plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_conv2_tc} -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-1} \
      -o $OUT/prof_${NCU_NAME:-conv2} $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 $OUT/ncu_full.log
fi
