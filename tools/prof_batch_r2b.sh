# the layouts of the sweep that had no capture of their own yet (same kernels as their twins, other strides)
for L in pbrt-align16 pbrt-soaos; do
  tools/profile.sh r2_c5_$(echo $L | tr - _) $L chrt2_kernel c5 > /dev/null 2>&1
done
for L in bvh8-align16 bvh8-q8-align16 bvh8-q16-align16 bvh8-q16-ci-align16 bvh8; do
  tools/profile.sh r2_c5_$(echo $L | tr - _) $L chrt8_kernel c5 > /dev/null 2>&1
done
tools/profile.sh r2_c4_pbrt_q16 pbrt-q16 cpq2_kernel c4 > /dev/null 2>&1
tools/profile.sh r2_c4_pbrt pbrt cpq2_kernel c4 > /dev/null 2>&1
rm -f gpurun_out/ncu_r2_c*.ncu-rep
ls gpurun_out/ncu_r2_c*.txt
