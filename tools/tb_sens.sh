#!/bin/bash
# Sensitivity of the T kernel to a 300-cycle busy wait in one role (diagnostic builds):
#   build:  for r in 0 1 2 3 4 5 6; do python -c "...build_profile_lib(name='libglassnet_s$r.so', defines=('GN_SENS=$r',))"; done
#   run:    tools/tb_sens.sh   (1 = issuer A per item, 2 = issuer B per item, 3 = E1 per item,
#           4 = E2 per item, 5 = loader per tile, 6 = psi per tile, 7 = issuer C per tile; 0 = none)
for r in 0 1 2 3 4 5 6 7; do
  GN_LIB=$PWD/paper_2405_19056_b200/libglassnet_s$r.so timeout 60 python tools/tb_time.py 2>&1 | grep T_B
done
