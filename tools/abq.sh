#!/bin/bash
# tools/abq.sh LAYOUT NAME... : closest-point (C4) throughput with the default library and each bin/libscion_NAME.so
L=$1; shift
run() { python bench.py --workload c4 --layout $L --no-e2e --no-cpu --sweep '' --steps 3 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('  %-18s %s %.1f %s' % (sys.argv[1], d['config'].get('layout'), d['value'], d['unit']))" $1; }
run default
for v in "$@"; do SCION_B200_LIB=$PWD/paper_2511_15028_b200/bin/libscion_$v.so run $v; done
