#!/bin/bash
# Build an A/B library variant: tools/build_variant.sh <out.so name> <git-rev|WORKTREE> [-DMACRO=...]
# (sources of csrc/ at that revision, compiled like build.py into paper_1410_2698_b200/<name>)
set -e
name=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_1410_2698_b200/csrc
if [[ $rev != WORKTREE ]]; then
  tmp=$(mktemp -d); git -C $root archive $rev paper_1410_2698_b200/csrc include | tar -x -C $tmp; src=$tmp/paper_1410_2698_b200/csrc
fi
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared \
    --expt-relaxed-constexpr -I$root/include "$@" -o $root/paper_1410_2698_b200/$name $src/*.cu
echo built $name
