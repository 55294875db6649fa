for L in sg-eq pbrt-soa dop14 identity pbrt-post ptr sg-eq-align16 pbrt-q16-soaos pbrt-soaos-align16; do
  tools/profile.sh r2_c5_$(echo $L | tr - _) $L chrt2_kernel c5 > /dev/null 2>&1
done
for L in bvh8-q8 bvh8-q16 bvh8-q16-ci bvh8-q8-ci-align16; do
  tools/profile.sh r2_c5_$(echo $L | tr - _) $L chrt8_kernel c5 > /dev/null 2>&1
done
tools/profile.sh r2_c3s_shared_slab shared-slab chrt2_kernel c3 "--scale 0.03125" > /dev/null 2>&1
ls -la gpurun_out/ncu_r2_c*.txt | wc -l
rm -f gpurun_out/ncu_r2_c*.ncu-rep
