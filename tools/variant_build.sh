#!/bin/bash
# Build a variant of _smes.so with extra nvcc defines for one source (experiments only):
#   tools/variant_build.sh NAME SRC.cu -DFOO=1 ...   -> build_var/_smes_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p build_var/$name
python paper_2602_09386_b200/build.py >/dev/null
objs=""
for f in paper_2602_09386_b200/build/*.o; do
  b=$(basename $f .o)
  if [ "$b.cu" == "$src" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr "$@" -c paper_2602_09386_b200/csrc/$src -o build_var/$name/$b.o
    objs="$objs build_var/$name/$b.o"
  else
    objs="$objs $f"
  fi
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static $objs -o build_var/_smes_$name.so
echo build_var/_smes_$name.so
