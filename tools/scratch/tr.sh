timeout 900 python -m pytest tests/test_gpu_train.py -q -x 2>&1 | tail -1
python tools/train_dp.py 20 256 paper bf16 2>&1 | tail -1
mkdir -p gpurun_out/tr2; ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr2/l.csv python tools/train_dp.py 3 256 paper bf16 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/tr2/l.csv 4
