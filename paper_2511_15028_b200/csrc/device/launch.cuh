// Kernel registry: one KernelEntry per layout, filled by the per-layout instantiation units
// (build/inst_<layout>.cu, stamped from device/inst.cu.in by the Makefile).
#pragma once
#include <cuda_runtime.h>

#include "scion_b200.h"
#include "scion_rt.cuh"

namespace scion {

struct LaunchArgs {
  TreeView view;
  const void* in;     // scion_ray* (closest_hit) or float* xyz (closest_point), device
  uint64_t n;
  void* out;          // scion_hit* or scion_cp*, device
  uint32_t* status;   // nullable
  scion_counters* counters;  // nullable => the counter-free kernel is launched
  unsigned long long* next;  // work-fetch counter, zeroed on the stream before launch
  cudaStream_t stream;
  int variant;
  int grid;           // 0 => occupancy * SM count
};

typedef cudaError_t (*launch_fn)(const LaunchArgs&);

struct CdScratch {  // device scratch of collision detection, cached by the owning tree between calls
  void* ptr = nullptr;
  size_t bytes = 0;
};
struct CdArgs {  // collision detection: two trees of the same layout on the same device
  TreeView a, b;
  scion_pair* out;
  uint64_t capacity;
  uint64_t frontier_capacity;
  uint64_t* out_count;      // host
  scion_cd_stats* stats;    // host, nullable
  cudaStream_t stream;
  CdScratch* scratch;
};
typedef cudaError_t (*cd_fn)(const CdArgs&, int* overflow_bits);
typedef cudaError_t (*occupancy_fn)(int* blocks_per_sm, int* regs, size_t* smem);
// builds the side treelet of the top levels (device/treelet.cuh) of a tree that is complete on the device: allocates
// *d_out (caller frees) and reports the slot count; synchronous
typedef cudaError_t (*treelet_fn)(const TreeView& view, uint8_t** d_out, uint32_t* slots);

struct KernelEntry {
  const char* layout;
  launch_fn closest_hit;
  launch_fn closest_point;  // null for 8-wide layouts (corpus.cpp:83)
  occupancy_fn hit_occupancy;
  cd_fn collide;  // null for 8-wide layouts (corpus.cpp:86)
  treelet_fn build_treelet;  // null unless the layout supports the staged top levels (traverse.cuh treelet_ok)
};

const KernelEntry* find_kernels(const char* layout);
int device_sm_count();

}  // namespace scion
