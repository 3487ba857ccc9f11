# Build libxpcs.so variants with extra -D flags: build/var/<name>/libxpcs.so (timing experiments; XPCS_LIB selects one)
# usage: bash tools/build_variants.sh name1 "-DFOO=1 -DBAR=2" name2 "-DFOO=2" ...
set -e
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  out=build/var/$name; mkdir -p $out
  objs=""
  for src in paper_2204_13241_b200/csrc/*.cu; do
    o=$out/$(basename $src .cu).o
    $NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude $defs -c $src -o $o &
    objs="$objs $o"
  done
  wait
  $NVCC $ARCH -shared -o $out/libxpcs.so $objs -lcudart -lcufft
  echo built $out/libxpcs.so
done
