#!/bin/bash
# tools/tl_probe.sh NAME... : treelet (variant 2) vs default kernel, identical-results check + timing, for the default
# library and each bin/libscion_NAME.so (tools/make_variant.sh)
echo "== default build"; python tools/gpu_probe.py --stage
for v in "$@"; do echo "== $v"; SCION_B200_LIB=$PWD/paper_2511_15028_b200/bin/libscion_$v.so python tools/gpu_probe.py --stage; done
