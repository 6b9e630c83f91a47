#!/usr/bin/env bash
# dev tool: variants of libxdg_b200.so with other multifrontal launch-bounds / loads-in-flight settings
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"; mkdir -p $ROOT/variants
build() { # name flags...
  name=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC -Xcompiler -O3 --threads 0 -Xlinker -soname=libxdg_b200.so -I $ROOT/include "$@" -o $ROOT/variants/lib_$name.so $ROOT/paper_2003_02431_b200/csrc/*.cu
}
build minb4_u8 -DMF_MINB=4 -DMF_U=8 &
build minb2_u8 -DMF_MINB=2 -DMF_U=8 &
build minb3_u6 -DMF_MINB=3 -DMF_U=6 &
build minb3_u12 -DMF_MINB=3 -DMF_U=12 &
wait
build minb4_u6 -DMF_MINB=4 -DMF_U=6 &
build minb2_u12 -DMF_MINB=2 -DMF_U=12 &
build minb2_u16 -DMF_MINB=2 -DMF_U=16 &
wait
ls -la $ROOT/variants/*.so
