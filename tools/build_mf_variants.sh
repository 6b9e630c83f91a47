#!/usr/bin/env bash
# dev tool: variants of libxdg_b200.so with other multifrontal launch-bounds / loads-in-flight settings
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"; mkdir -p $ROOT/variants
build() { # name flags...
  name=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC -Xcompiler -O3 --threads 0 -Xlinker -soname=libxdg_b200.so -I $ROOT/include "$@" -o $ROOT/variants/lib_$name.so $ROOT/paper_2003_02431_b200/csrc/*.cu
}
if [ "${1:-}" = "count" ]; then  # candidates for the cfg2 GMRES iteration-count check
build mr4_mu8_minb2 -DMF_MR=4 -DMF_MU=8 -DMF_MINB=2 &
build mr4_mu12_minb2 -DMF_MR=4 -DMF_MU=12 -DMF_MINB=2 &
build mr3_mu10_minb2 -DMF_MR=3 -DMF_MU=10 -DMF_MINB=2 &
build mr3_mu6_minb2 -DMF_MR=3 -DMF_MU=6 -DMF_MINB=2 &
wait
build mr3_mu12_minb2 -DMF_MR=3 -DMF_MU=12 -DMF_MINB=2 &
build mr2_mu8_minb2 -DMF_MR=2 -DMF_MU=8 -DMF_MINB=2 &
build mr2_mu8_minb3 -DMF_MR=2 -DMF_MU=8 -DMF_MINB=3 &
wait
ls -la $ROOT/variants/*.so
exit 0
fi
if [ "${1:-}" = "mr3" ]; then
build mr3_mu8_minb2 -DMF_MR=3 -DMF_MU=8 -DMF_MINB=2 &
build mr3_mu12_minb2 -DMF_MR=3 -DMF_MU=12 -DMF_MINB=2 &
build mr3_mu6_minb2 -DMF_MR=3 -DMF_MU=6 -DMF_MINB=2 &
build mr3_mu10_minb2 -DMF_MR=3 -DMF_MU=10 -DMF_MINB=2 &
wait
build mr3_mu8_minb3 -DMF_MR=3 -DMF_MU=8 -DMF_MINB=3 &
build mr5_mu6_minb2 -DMF_MR=5 -DMF_MU=6 -DMF_MINB=2 &
build mr6_mu6_minb2 -DMF_MR=6 -DMF_MU=6 -DMF_MINB=2 &
wait
ls -la $ROOT/variants/*.so
exit 0
fi
if [ "${1:-}" = "mr" ]; then
build mr2_mu12 -DMF_MR=2 -DMF_MU=12 &
build mr2_mu16_minb2 -DMF_MR=2 -DMF_MU=16 -DMF_MINB=2 &
build mr4_mu8_minb2 -DMF_MR=4 -DMF_MU=8 -DMF_MINB=2 &
build mr4_mu4 -DMF_MR=4 -DMF_MU=4 &
wait
build mr1_mu16 -DMF_MR=1 -DMF_MU=16 &
build mr4_mu12_minb2 -DMF_MR=4 -DMF_MU=12 -DMF_MINB=2 &
build mr2_mu6 -DMF_MR=2 -DMF_MU=6 &
build mr3_mu8_minb2 -DMF_MR=3 -DMF_MU=8 -DMF_MINB=2 &
wait
ls -la $ROOT/variants/*.so
exit 0
fi
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
