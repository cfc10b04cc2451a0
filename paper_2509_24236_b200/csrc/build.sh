#!/bin/sh
# Builds libpft.so for sm_100a (B200).  Used by __graft_entry__.build() and by hand.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
OUT=${1:-$HERE/../libpft.so}
if [ $# -gt 0 ]; then shift; fi
EXTRA="$@"
NCCL_INC=$(python -c 'import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], "include"))')
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Xptxas -v $EXTRA -I"$NCCL_INC" \
  "$HERE/volume.cu" "$HERE/integrate.cu" "$HERE/track.cu" "$HERE/extract.cu" "$HERE/abi.cu" \
  -o "$OUT.tmp" -ldl 2> "$HERE/../ptxas.log" || { cat "$HERE/../ptxas.log"; exit 1; }
mv "$OUT.tmp" "$OUT"
