#!/bin/bash
# tools/ab_parity.sh LAYOUTS NAME... : for each variant library bin/libscion_NAME.so — bit-exactness against the oracle (the parity
# tests run on the variant) and the C5 probe timing next to the default library
L=$1; shift
for v in "$@"; do echo "== parity $v"; SCION_B200_LIB=$PWD/paper_2511_15028_b200/bin/libscion_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "closest_hit_matches_oracle or closest_point_matches_oracle or edge_cases or golden" 2>&1 | tail -2; done
echo "== timing"; tools/ab.sh $L "$@"
