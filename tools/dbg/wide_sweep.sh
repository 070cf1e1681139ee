#!/bin/bash
# A/B of the wide pooling kernel: ring depth (alternative build) x tiles per CTA
for lib in paper_2310_05218_b200/libslideconv_b200.so tools/dbg/lib_nb4.so; do
  for tpc in 1 2 4 8; do
    echo "== $lib tpc=$tpc"
    SLIDECONV_B200_LIB=$lib SC_WIDE_TPC=$tpc python tools/dbg/wide_ab.py 2>&1 | head -3
  done
done
