set -u
OUT=gpurun_out/r02y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
DI_NVCC_EXTRA="-DDI_C3R_NSL=16 -DDI_C3R_PF=24" DI_EXP_NAME=nsl16 python paper_1701_03891_b200/build.py > $OUT/b1.log 2>&1 || echo B1 FAILED
DI_NVCC_EXTRA="-DDI_C3R_PF=40" DI_EXP_NAME=pf40 python paper_1701_03891_b200/build.py > $OUT/b2.log 2>&1 || echo B2 FAILED
DI_NVCC_EXTRA="-DDI_C3R_NSL=16 -DDI_C3R_PF=24 -DDI_PROF_CONV3" DI_EXP_NAME=nsl16p python paper_1701_03891_b200/build.py > $OUT/b3.log 2>&1 || echo B3 FAILED
bash tools/scratch/ab_lib.sh 3 product nsl16 pf40
DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_nsl16p.so timeout 300 python tools/time_stages.py lowrate 3 2>&1 | tail -3
