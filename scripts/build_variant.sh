#!/bin/bash
# build a variant of the library with extra nvcc flags into paper_variants/<name>/
# (design experiments; time it with PB_ROOT=paper_variants/<name>)
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
dst=$ROOT/paper_variants/$name
rm -rf $dst; mkdir -p $dst
cp -r $ROOT/paper_2503_19894_b200 $dst/
rm -rf $dst/paper_2503_19894_b200/csrc/build $dst/paper_2503_19894_b200/jit_cache
make -s -j8 -C $dst/paper_2503_19894_b200/csrc NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off -I$ROOT/include -I$dst/paper_2503_19894_b200/csrc $*" ROOT=$ROOT > /dev/null
echo "built $dst"
