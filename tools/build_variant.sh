#!/bin/bash
# Build an experimental libxpcs variant with extra -D flags (timing experiments only; load it with XPCS_LIB=...).
#   tools/build_variant.sh NAME "-DXPCS_I8_GROUPS=2 -DXPCS_I8_STAGES=6"
set -e
cd "$(dirname "$0")/.."
name=$1; shift
flags="$*"
mkdir -p build/var_$name
objs=""
for f in paper_2204_13241_b200/csrc/*.cu; do
  b=$(basename "$f" .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
       --expt-relaxed-constexpr -Iinclude $flags -c "$f" -o build/var_$name/$b.o > /dev/null 2>&1 &
  objs="$objs build/var_$name/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/libxpcs_$name.so $objs -lcudart -lcufft
echo build/libxpcs_$name.so
