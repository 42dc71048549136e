#!/bin/bash
# Experiment (tools/): build replay.cu tuning variants of the library into
# build/variants/<name>.so (the other translation units compiled once), so one
# gpurun call can time them by swapping the .so in place.
# usage: tools/build_variants.sh name1="-DFOO=1 -DBAR=2" name2="..."
set -e
cd "$(dirname "$0")/.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xptxas -O3"
C=paper_2512_18725_b200/csrc
mkdir -p build/variants build/obj
for f in common csv predict rows; do
  [ build/obj/$f.o -nt $C/$f.cu ] || nvcc $ARCH $FLAGS -c $C/$f.cu -o build/obj/$f.o &
done
wait
for spec in "$@"; do
  name="${spec%%=*}"; defs="${spec#*=}"
  ( nvcc $ARCH $FLAGS $defs -c $C/replay.cu -o build/obj/replay_$name.o &&
    nvcc $ARCH -shared -o build/variants/$name.so build/obj/{common,csv,predict,rows}.o build/obj/replay_$name.o &&
    echo "built $name ($defs)" ) &
done
wait
