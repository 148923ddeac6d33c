#!/bin/bash
# Build an in-tree library variant paper_1704_03767_b200/libtaub200_<tag>.so whose <file>.cu comes from git
# revision <rev> (WORKTREE: the working tree; every other object from the current build), compiled with
# optional extra nvcc flags, for TB_LIB_VARIANT A/B runs.
#   tools/build_variant.sh <tag> <rev> <file.cu> [nvcc flags...]
set -e
tag=$1; rev=$2; f=$3; shift 3; extra="$*"
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_1704_03767_b200/csrc
make -s -C "$csrc"
tmp=$(mktemp -d)
if [ "$rev" = WORKTREE ]; then cp "$csrc/$f" "$csrc/_variant_$f"; else git -C "$root" show "$rev:paper_1704_03767_b200/csrc/$f" > "$csrc/_variant_$f"; fi
objs=""
for o in "$csrc"/_build/*.o; do
  b=$(basename "$o" .o)
  if [ "$b.cu" = "$f" ]; then continue; fi
  objs="$objs $o"
done
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $extra -I"$csrc" -c "$csrc/_variant_$f" -o "$tmp/v.o"
$NV $ARCH -shared -o "$root/paper_1704_03767_b200/libtaub200_$tag.so" $objs "$tmp/v.o" -cudart static
rm -rf "$tmp" "$csrc/_variant_$f"
echo "built paper_1704_03767_b200/libtaub200_$tag.so ($f from $rev $extra)"
