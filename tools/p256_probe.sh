for v in tri256 cover256 both256; do echo "== parity $v"; SCION_B200_LIB=$PWD/paper_2511_15028_b200/bin/libscion_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "closest_hit_matches_oracle or closest_point_matches_oracle or edge_cases" 2>&1 | tail -2; done
echo "== timing"; tools/ab.sh pbrt-q16,pbrt,bvh8-q8-ci,sg-eq,pbrt-soa tri256
tools/ab.sh identity,pbrt-post cover256 both256
