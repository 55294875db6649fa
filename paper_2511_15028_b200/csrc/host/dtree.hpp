// Device-resident PhysicalTree: the packed image, its header, the per-launch work-counter pool and the
// staging state of the host entry points.  Shared by abi.cu (queries) and comm.cu (replication over NCCL).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "../device/launch.cuh"
#include "physical.hpp"
#include "scion_b200.h"

namespace scion {

// ------------------------------------------------------------------ device image
// One contiguous allocation: [ImageHeader | buffer 0 | buffer 1 | ...], every buffer 256-byte
// aligned and followed by >= 16 bytes of slack (covering vector loads, geometry.cuh).
constexpr uint64_t kImageMagic = 0x3130304d49434353ull;  // "SCCIM001"
struct ImageHeader {
  uint64_t magic;
  uint64_t total_bytes;
  char layout[48];
  int32_t nbuf, nglob;
  uint64_t offset[SCION_MAX_BUFFERS];
  uint64_t bytes[SCION_MAX_BUFFERS];
  uint64_t count[SCION_MAX_BUFFERS];
  uint64_t seg_base[SCION_MAX_BUFFERS][SCION_MAX_SEGMENTS];
  uint32_t glob[SCION_MAX_GLOBALS][4];
  uint64_t root0;
  float carried[6];
  uint64_t nprims;
  uint8_t pad[16];
};
static_assert(sizeof(ImageHeader) % 16 == 0, "image header must keep 16-byte alignment");
constexpr uint64_t kHeaderBytes = (sizeof(ImageHeader) + 255) / 256 * 256;
constexpr int kCounterBlock = 64;  // work-fetch counters are allocated in blocks of this many

// One work-fetch counter per LAUNCH IN FLIGHT.  A slot is handed out again only after the event
// recorded behind the launch that used it has completed, so no launch — on any stream, from any host
// thread — can zero or share the counter of a kernel that is still running; the pool grows when every
// slot is busy (concurrent queries on a shared immutable tree).
struct CounterSlot {
  unsigned long long* ctr = nullptr;
  cudaEvent_t done = nullptr;  // recorded on the launch stream right behind the kernel
  bool pending = false;        // handed out, event not recorded yet
};
struct CounterPool {
  std::mutex mu;
  std::vector<CounterSlot> slots;
  std::vector<void*> blocks;
  size_t cursor = 0;
  cudaError_t grow() {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, kCounterBlock * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    blocks.push_back(p);
    for (int i = 0; i < kCounterBlock; i++) {
      CounterSlot s;
      s.ctr = (unsigned long long*)p + i;
      e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
      slots.push_back(s);
    }
    return cudaSuccess;
  }
  // index of a slot no live kernel uses; marks it pending
  cudaError_t take(size_t* out, unsigned long long** ctr) {
    std::lock_guard<std::mutex> lock(mu);
    for (int pass = 0; pass < 2; pass++) {
      const size_t n = slots.size();
      for (size_t k = 0; k < n; k++) {
        const size_t i = (cursor + k) % n;
        CounterSlot& s = slots[i];
        if (s.pending) continue;
        const cudaError_t q = cudaEventQuery(s.done);
        if (q == cudaSuccess) {
          s.pending = true;
          cursor = (i + 1) % n;
          *out = i;
          *ctr = s.ctr;
          return cudaSuccess;
        }
        if (q != cudaErrorNotReady) return q;
      }
      cursor = n;  // first slot of the new block
      const cudaError_t e = grow();
      if (e != cudaSuccess) return e;
    }
    return cudaErrorUnknown;
  }
  // the launch (or its failure) is behind us: record the guard event on its stream
  cudaError_t release(size_t i, cudaStream_t stream, bool launched) {
    std::lock_guard<std::mutex> lock(mu);
    cudaError_t e = launched ? cudaEventRecord(slots[i].done, stream) : cudaSuccess;
    slots[i].pending = false;
    return e;
  }
  void destroy() {
    for (auto& s : slots) if (s.done) cudaEventDestroy(s.done);
    for (void* p : blocks) cudaFree(p);
    slots.clear();
    blocks.clear();
  }
};


}  // namespace scion

struct scion_dtree {
  const scion::LayoutEntry* layout = nullptr;
  const scion::KernelEntry* kernels = nullptr;
  int device = 0;
  uint8_t* image = nullptr;
  bool owns_image = true;
  scion::ImageHeader header{};
  scion::TreeView view{};
  uint8_t* treelet = nullptr;  // side treelet of the top levels (device/treelet.cuh), built once in finish_dtree; a cache, not part of the image
  scion::CounterPool counters;  // one work-fetch counter per launch in flight
  // staging for the host entry points
  static constexpr int kSlots = 4;  // staging slots of the host entry points: H2D(k+1) || kernel(k) || D2H(k-1)
  void* h2d[kSlots] = {};
  void* d2h[kSlots] = {};
  void* pk[kSlots] = {};  // packed-ray staging (scion_closest_hit_host_packed), allocated on first use
  uint64_t pk_chunk = 0;
  uint32_t* d_status[kSlots] = {};
  cudaStream_t streams[kSlots] = {};  // [0] uploads, [1] and [2] kernels (alternating), [3] downloads
  cudaEvent_t ev_in[kSlots] = {}, ev_run[kSlots] = {}, ev_out[kSlots] = {};
  uint64_t chunk = 0;
  scion::CdScratch cd_scratch;  // collision detection frontiers (guarded by host_mutex)
  std::mutex host_mutex;
};


namespace scion {
// rebuilds the by-value kernel view from t.header / t.image
void fill_view(scion_dtree& t);
// kernels + first counter block + view; returns a scion_status (message via scion_last_error)
int finish_dtree(scion_dtree* t);
int abi_fail(int code, const std::string& msg);
}  // namespace scion
