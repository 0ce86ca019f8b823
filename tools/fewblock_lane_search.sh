#!/bin/bash
# Which output lanes of hash_fewblock_kernel should be stored from copies (kCopyLanes in
# csrc/kernel_fewblock.cu)?  Compiles the kernel file with random lane sets and counts, with
# tools/sass_bank_census.py, the LOP3 / SHF of the round loop whose three sources share a register
# bank -- for the four shapes that store output blocks inside the loop.  No GPU needed; ~5 s per set.
# usage: bash tools/fewblock_lane_search.sh [candidates (default 36)]
cd "$(dirname "$0")/../paper_1902_05320_b200/csrc" || exit 1
N=${1:-36}
for i in $(seq 1 "$N"); do
  mask=$(python3 -c "import random; random.seed($i); print(hex(random.getrandbits(21)))")
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 "-DB200SHA3_FEWBLOCK_COPY_LANES=${mask}u" \
       -c -o /tmp/fewblock_search.o kernel_fewblock.cu 2>/dev/null || continue
  echo "$mask: $(python3 ../../tools/sass_bank_census.py /tmp/fewblock_search.o | grep -E 'fewblock_kernel<(17|21), 8, (64|128)>' \
       | awk -F'|' '{printf "%s ", $4}')"
done | sort -t: -k2
