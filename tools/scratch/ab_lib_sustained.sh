# alternate libraries (product + experiment builds named by DI_EXP_NAME) in separate processes, 3 rounds
# usage: bash tools/scratch/ab_lib_sustained.sh name1 name2 ...   (libdeepinverse_exp_<name>.so)
for r in 1 2 3; do
  DI_LIB=paper_1701_03891_b200/libdeepinverse.so python tools/scratch/sustained_one.py
  for n in "$@"; do DI_LIB=paper_1701_03891_b200/libdeepinverse_exp_$n.so python tools/scratch/sustained_one.py; done
done
