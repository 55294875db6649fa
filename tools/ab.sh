#!/bin/bash
# tools/ab.sh LAYOUTS NAME... : time the C5 probe with the default library and each bin/libscion_NAME.so
L=$1; shift
python tools/gpu_probe.py --c5 $L
for v in "$@"; do SCION_B200_LIB=$PWD/paper_2511_15028_b200/bin/libscion_$v.so python tools/gpu_probe.py --c5 $L; done
