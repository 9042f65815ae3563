#!/usr/bin/env bash
out=gpurun_out/${1:-plink}; mkdir -p $out
for cfg in "32768 4 1" "32768 4 0" "32768 3 0" "16384 8 1" "16384 8 0" "65536 4 1" "8192 8 1"; do
  set -- $cfg
  COLOC_STAGING_CHUNK_KB=$1 COLOC_STAGING_RING=$2 COLOC_STAGING_H2D_NT=$3 timeout 120 python tools/dbg/pageable_link.py >> $out/sweep.jsonl 2>&1
done
