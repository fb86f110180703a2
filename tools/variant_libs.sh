#!/bin/bash
# Builds variant copies of the library that differ in one translation unit's
# -D flags, for A/B runs on the GPU box (FLEXMARL_LIB=<variant> python bench.py ...).
#   tools/variant_libs.sh k_band.cu s16b24 "-DFM_STATS_STAGES=16 -DFM_BAND_STAGES=24" ...
set -e
cd "$(dirname "$0")/.."
python -c "import paper_2602_09578_b200.build as b; b.build()" > /dev/null
SRC=$1; shift
OUT=paper_2602_09578_b200/_native/variants
mkdir -p $OUT
NCCL=$(python -c "import paper_2602_09578_b200.build as b; print(b.nccl_dir() or '')")
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  objs=""
  for o in build/obj/*.o; do
    if [ "$(basename $o)" = "$SRC.o" ]; then
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
        -Iinclude -Ipaper_2602_09578_b200/csrc ${NCCL:+-I$NCCL/include} $defs -c paper_2602_09578_b200/csrc/$SRC -o /tmp/var_$name.o
      objs="$objs /tmp/var_$name.o"
    else
      objs="$objs $o"
    fi
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so $objs ${NCCL:+-L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib}
  echo "$OUT/lib_$name.so"
done
