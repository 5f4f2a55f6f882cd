# conv1 phase-stacked form (conflict-free staging): parity and A/B stage times against the plain .ws M = 64 form
set -u
OUT=gpurun_out/r06c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_elementwise.py -m gpu -x -q > $OUT/pytest_elem.log 2>&1; echo "elem rc=$?"; tail -15 $OUT/pytest_elem.log
for i in 1 2 3; do
  timeout 300 python tools/time_stages.py lowrate 20 >> $OUT/stages_ph.jsonl 2>&1
  DI_EXP_C1_PLAIN=1 timeout 300 python tools/time_stages.py lowrate 20 >> $OUT/stages_plain.jsonl 2>&1
done
grep -h stages_ms $OUT/stages_ph.jsonl | cut -c1-160; echo plain; grep -h stages_ms $OUT/stages_plain.jsonl | cut -c1-160
