#!/bin/bash
# A/B timing of T-kernel variants in one GPU session: ab_time.sh LIB1 LIB2 ... (names under
# paper_2405_19056_b200/), interleaved, 3 rounds (tools/tb_time.py: c3 x 8 frames).
for r in 1 2 3; do
  for L in "$@"; do
    GN_LIB=$PWD/paper_2405_19056_b200/$L python tools/tb_time.py 2>&1 | grep T_B
  done
done
