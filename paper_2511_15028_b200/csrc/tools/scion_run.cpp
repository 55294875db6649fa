// scion_run — native C++ harness over the C ABI (include/scion_b200.h): the slice of the reference CLI
// (`layoutc footprint | bench`) that belongs to the traversal path, written the way a
// maintainer of the C++ reference would call the B200 backend — nothing here but the C ABI and the
// CUDA runtime (device buffers, events).
//   scion_run layouts
//   scion_run footprint <layout> <terrain|sphere|cloud>:<N>
//   scion_run bench     <layout> <scene>:<N> <queries> [primary|secondary|points] [--host-encode] [--gpus G]
// `--gpus G` (G > 1): ONE process drives G devices — ncclCommInitAll, the tree encoded on device 0 and replicated with
// one ncclBroadcast (scion_dtree_broadcast_all), queries partitioned contiguously (scion_partition) and generated on
// each device from (seed, global index), results gathered by query index (scion_gather_results_all); n_gpus = G in the row.
// `bench` follows the paper's protocol: 1 warm-up + 9 runs, drop the 2
// lowest and 2 highest, mean of the remaining 5; prints one CSV row; the un-timed instrumented pass gives
// the reference's counters (node visits, primitive tests) and the algorithmic bytes per query.
// Exit codes as the reference CLI: 0 pass, 1 diagnostics / query errors, 2 usage.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "scion_b200.h"

static int die(int code, const char* what) {
  std::fprintf(stderr, "scion_run: %s: %s\n", what, scion_last_error());
  return code;
}
#define CK(x) do { if ((x) != SCION_OK) return die(1, #x); } while (0)
#define CU(x) do { cudaError_t e__ = (x); if (e__ != cudaSuccess) { std::fprintf(stderr, "scion_run: %s: %s\n", #x, cudaGetErrorString(e__)); return 1; } } while (0)

static int make_scene(const std::string& spec, scion_scene** out, bool* terrain) {
  const size_t c = spec.find(':');
  const std::string kind = spec.substr(0, c);
  const uint64_t n = c == std::string::npos ? 64 : std::strtoull(spec.c_str() + c + 1, nullptr, 10);
  *terrain = kind == "terrain";
  if (kind == "terrain") return scion_scene_terrain((uint32_t)n, 1, out);
  if (kind == "sphere") return scion_scene_sphere((uint32_t)n, 1, out);
  if (kind == "cloud") return scion_scene_cloud(n, 1, out);
  return SCION_ERR_ARG;
}

// ---- multi-GPU bench (single process, G devices): SURVEY §8e
static int bench_multi(int G, scion_dtree* dt0, const scion_layout_info& li, const char* layout, const char* scene_spec, uint64_t n, const std::string& kind, bool terrain,
                       const float lo[3], const float hi[3], uint64_t node_bytes, uint64_t nprims) {
  const bool cpq = kind == "points";
  const uint32_t q_sz = cpq ? 12 : (uint32_t)sizeof(scion_ray), r_sz = cpq ? (uint32_t)sizeof(scion_cp) : (uint32_t)sizeof(scion_hit);
  std::vector<scion_comm*> comms((size_t)G, nullptr);
  CK(scion_comm_init_all(G, nullptr, comms.data()));
  std::vector<scion_dtree*> trees((size_t)G, nullptr);
  cudaEvent_t b0, b1;
  CU(cudaSetDevice(0));
  CU(cudaEventCreate(&b0));
  CU(cudaEventCreate(&b1));
  CU(cudaEventRecord(b0));
  CK(scion_dtree_broadcast_all(dt0, 0, comms.data(), G, nullptr, trees.data()));
  CU(cudaSetDevice(0));
  CU(cudaEventRecord(b1));
  CU(cudaEventSynchronize(b1));
  float bcast_ms = 0;
  CU(cudaEventElapsedTime(&bcast_ms, b0, b1));
  std::vector<void*> d_q((size_t)G), d_r((size_t)G), d_full((size_t)G);
  std::vector<uint64_t> first((size_t)G), count((size_t)G);
  std::vector<cudaEvent_t> e0((size_t)G), e1((size_t)G);
  uint32_t side = 1;
  while ((uint64_t)(side + 1) * (side + 1) <= n) side++;
  scion_camera cam;
  scion_camera_default(lo, hi, terrain ? 1 : 0, side, side, &cam);
  for (int g = 0; g < G; g++) {
    CU(cudaSetDevice(g));
    scion_partition(n, g, G, &first[(size_t)g], &count[(size_t)g]);
    CU(cudaMalloc(&d_q[(size_t)g], (count[(size_t)g] + 1) * q_sz));
    CU(cudaMalloc(&d_full[(size_t)g], (n + 1) * r_sz));
    d_r[(size_t)g] = (uint8_t*)d_full[(size_t)g] + first[(size_t)g] * r_sz;  // results land in place: the gather moves only the other ranks' slices
    CU(cudaEventCreate(&e0[(size_t)g]));
    CU(cudaEventCreate(&e1[(size_t)g]));
    if (cpq) CK(scion_gen_points(lo, hi, 7, first[(size_t)g], count[(size_t)g], (float*)d_q[(size_t)g], nullptr));
    else if (kind == "secondary") CK(scion_gen_secondary(trees[(size_t)g], 7, first[(size_t)g], count[(size_t)g], (scion_ray*)d_q[(size_t)g], nullptr));
    else CK(scion_gen_primary(&cam, first[(size_t)g], count[(size_t)g], (scion_ray*)d_q[(size_t)g], nullptr));
  }
  std::vector<float> ms;
  for (int it = 0; it < 10; it++) {
    for (int g = 0; g < G; g++) {
      CU(cudaSetDevice(g));
      CU(cudaEventRecord(e0[(size_t)g]));
      if (cpq) CK(scion_closest_point(trees[(size_t)g], (const float*)d_q[(size_t)g], count[(size_t)g], (scion_cp*)d_r[(size_t)g], nullptr, nullptr, 0, nullptr));
      else CK(scion_closest_hit(trees[(size_t)g], (const scion_ray*)d_q[(size_t)g], count[(size_t)g], (scion_hit*)d_r[(size_t)g], nullptr, nullptr, 0, nullptr));
      CU(cudaEventRecord(e1[(size_t)g]));
    }
    float worst = 0;
    for (int g = 0; g < G; g++) {
      CU(cudaSetDevice(g));
      CU(cudaEventSynchronize(e1[(size_t)g]));
      float t = 0;
      CU(cudaEventElapsedTime(&t, e0[(size_t)g], e1[(size_t)g]));
      worst = std::max(worst, t);
    }
    if (it) ms.push_back(worst);  // max over devices
  }
  std::sort(ms.begin(), ms.end());
  const double mean_ms = (ms[2] + ms[3] + ms[4] + ms[5] + ms[6]) / 5.0;
  CU(cudaSetDevice(0));
  CU(cudaEventRecord(b0));
  CK(scion_gather_results_all(comms.data(), G, d_r.data(), n, r_sz, d_full.data(), nullptr));
  for (int g = 0; g < G; g++) { CU(cudaSetDevice(g)); CU(cudaDeviceSynchronize()); }
  CU(cudaSetDevice(0));
  CU(cudaEventRecord(b1));
  CU(cudaEventSynchronize(b1));
  float gather_ms = 0;
  CU(cudaEventElapsedTime(&gather_ms, b0, b1));
  // every device must now hold the same n records
  std::vector<uint8_t> ref((size_t)n * r_sz), other((size_t)n * r_sz);
  CU(cudaMemcpy(ref.data(), d_full[0], ref.size(), cudaMemcpyDeviceToHost));
  int mismatched = 0;
  for (int g = 1; g < G; g++) {
    CU(cudaSetDevice(g));
    CU(cudaMemcpy(other.data(), d_full[(size_t)g], other.size(), cudaMemcpyDeviceToHost));
    mismatched += std::memcmp(ref.data(), other.data(), ref.size()) != 0;
  }
  std::printf("layout,algorithm,scene,n_gpus,queries,kind,mean_ms,mqueries_per_s,bvh_bytes_per_prim,broadcast_ms,gather_ms,gather_mismatches\n");
  std::printf("%s,%s,%s,%d,%llu,%s,%.4f,%.2f,%.3f,%.3f,%.3f,%d\n", layout, cpq ? "cpq" : "chrt", scene_spec, G, (unsigned long long)n, kind.c_str(), mean_ms, (double)n / mean_ms / 1e3,
              (double)node_bytes / (double)nprims, bcast_ms, gather_ms, mismatched);
  for (int g = 0; g < G; g++) {
    cudaSetDevice(g);
    cudaFree(d_q[(size_t)g]); cudaFree(d_full[(size_t)g]);
    if (g) scion_dtree_free(trees[(size_t)g]);
    scion_comm_free(comms[(size_t)g]);
  }
  (void)li;
  return mismatched ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: scion_run layouts | footprint <layout> <scene>:<N> | bench <layout> <scene>:<N> <queries> [primary|secondary|points] [--host-encode] [--gpus G] [--layout-file FILE.scion]\n");
    return 2;
  }
  // --layout-file FILE.scion (anywhere on the command line, repeatable): compile the file at run time and register it
  // under its stem (my_layout.scion -> my-layout) before the command runs — scion_layout_register, needs nvcc
  for (int i = 1; i + 1 < argc;) {
    if (std::strcmp(argv[i], "--layout-file") != 0) { i++; continue; }
    std::string path = argv[i + 1], name = path;
    const size_t slash = name.rfind('/');
    if (slash != std::string::npos) name = name.substr(slash + 1);
    const size_t dot = name.rfind('.');
    if (dot != std::string::npos) name = name.substr(0, dot);
    for (auto& c : name) if (c == '_') c = '-';
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) { std::fprintf(stderr, "scion_run: cannot read %s\n", path.c_str()); return 2; }
    std::string text;
    char buf[4096];
    for (size_t k; (k = std::fread(buf, 1, sizeof buf, f)) > 0;) text.append(buf, k);
    std::fclose(f);
    if (scion_layout_register(name.c_str(), text.c_str(), nullptr, nullptr) != SCION_OK) return die(1, "layout registration failed");
    std::fprintf(stderr, "registered layout '%s' from %s\n", name.c_str(), path.c_str());
    for (int k = i; k + 2 < argc; k++) argv[k] = argv[k + 2];  // drop the two arguments
    argc -= 2;
  }
  if (argc < 2) return 2;
  const std::string cmd = argv[1];
  if (cmd == "layouts") {
    for (int i = 0; i < scion_layout_count(); i++) {
      scion_layout_info li;
      CK(scion_layout_info_at(i, &li));
      std::printf("%-14s family=%d arity=%d node_stride=%u segments=%u ref_bits=%u max_leaf=%u cpq=%d\n", li.name, li.family, li.arity, li.node_stride, li.n_segments, li.ref_bits,
                  li.max_leaf, li.has_cpq);
    }
    return 0;
  }
  if ((cmd != "footprint" && cmd != "bench") || argc < 4) return 2;
  const char* layout = argv[2];
  scion_layout_info li;
  if (scion_layout_find(layout, &li) != SCION_OK) return die(2, "unknown layout");
  scion_scene* scene = nullptr;
  bool terrain = false;
  if (make_scene(argv[3], &scene, &terrain) != SCION_OK) return die(2, "bad scene");
  scion_ltree* lt = nullptr;
  CK(scion_build_sah(scene, 32, 4, 64, &lt));
  if (li.arity == 8) CK(scion_ltree_collapse8(lt));
  const uint64_t nprims = scion_ltree_nprims(lt);

  if (cmd == "footprint") {
    scion_ptree* pt = nullptr;
    CK(scion_encode(lt, layout, &pt));
    std::printf("{\"layout\": \"%s\", \"scene\": \"%s\", \"primitives\": %llu, \"total_bytes\": %llu, \"node_bytes\": %llu, \"bvh_bytes_per_prim\": %.6f, \"node_stride\": %u}\n", layout,
                argv[3], (unsigned long long)nprims, (unsigned long long)scion_ptree_total_bytes(pt), (unsigned long long)scion_ptree_node_bytes(pt),
                (double)scion_ptree_node_bytes(pt) / (double)nprims, li.node_stride);
    scion_ptree_free(pt);
    scion_ltree_free(lt);
    scion_scene_free(scene);
    return 0;
  }

  if (argc < 5) return 2;
  const uint64_t n = std::strtoull(argv[4], nullptr, 10);
  std::string kind = argc > 5 && argv[5][0] != '-' ? argv[5] : "primary";
  bool host_encode = false;
  int gpus = 1;
  for (int i = 5; i < argc; i++) {
    host_encode |= std::strcmp(argv[i], "--host-encode") == 0;
    if (std::strcmp(argv[i], "--gpus") == 0 && i + 1 < argc) gpus = std::atoi(argv[i + 1]);
  }
  if (gpus < 1) return 2;
  int ndev = 0;
  if (scion_device_count(&ndev) != SCION_OK) return die(1, "no CUDA device");
  if (gpus > ndev) { std::fprintf(stderr, "scion_run: --gpus %d but this node exposes %d CUDA device(s)\n", gpus, ndev); return 2; }
  const bool cpq = kind == "points";
  if (cpq && !li.has_cpq) { std::fprintf(stderr, "scion_run: cpq requires a binary layout\n"); return 2; }

  scion_dtree* dt = nullptr;
  uint64_t node_bytes = 0;
  double hot = (double)li.node_stride;  // bytes of the segment every visit reads (segment 0 of the node group)
  {
    scion_ptree* pt = nullptr;  // footprint numbers come from the host plan either way
    CK(scion_encode(lt, layout, &pt));
    node_bytes = scion_ptree_node_bytes(pt);
    for (int b = 0; b < scion_ptree_nbuffers(pt) && li.n_segments > 1; b++) {
      uint64_t bases[8], count = 0;
      const int ns = scion_ptree_segment_bases(pt, b, bases, 8);
      CK(scion_ptree_buffer(pt, b, nullptr, nullptr, nullptr, &count));
      if (ns > 1 && count) hot = (double)(bases[1] - bases[0]) / (double)count;  // plan.cpp:333-347: base[s+1] = base[s] + count * stride[s] (aligned)
    }
    if (host_encode) CK(scion_dtree_upload(pt, 0, &dt));
    scion_ptree_free(pt);
    if (!host_encode) CK(scion_encode_device(lt, layout, 0, &dt));  // build_physical on the GPU
  }
  float lo[3], hi[3];
  scion_scene_bounds(scene, lo, hi);
  if (gpus > 1 || std::getenv("SCION_RUN_FORCE_MULTI")) {  // the env switch drives the same code over a 1-device communicator (tests on a 1-GPU box)
    const int rc = bench_multi(gpus, dt, li, layout, argv[3], n, kind, terrain, lo, hi, node_bytes, nprims);
    scion_dtree_free(dt);
    scion_ltree_free(lt);
    scion_scene_free(scene);
    return rc;
  }
  void *d_q = nullptr, *d_r = nullptr;
  uint32_t* d_st = nullptr;
  scion_counters* d_ctr = nullptr;
  CU(cudaMalloc(&d_q, n * (cpq ? 12 : sizeof(scion_ray))));
  CU(cudaMalloc(&d_r, n * (cpq ? sizeof(scion_cp) : sizeof(scion_hit))));
  CU(cudaMalloc(&d_st, n * sizeof(uint32_t)));
  CU(cudaMalloc(&d_ctr, n * sizeof(scion_counters)));
  if (cpq) {
    CK(scion_gen_points(lo, hi, 7, 0, n, (float*)d_q, nullptr));
  } else if (kind == "secondary") {
    CK(scion_gen_secondary(dt, 7, 0, n, (scion_ray*)d_q, nullptr));
  } else {
    uint32_t side = 1;
    while ((uint64_t)(side + 1) * (side + 1) <= n) side++;
    scion_camera cam;
    scion_camera_default(lo, hi, terrain ? 1 : 0, side, side, &cam);
    CK(scion_gen_primary(&cam, 0, n, (scion_ray*)d_q, nullptr));
  }
  auto run = [&](uint32_t* st, scion_counters* ctr) {
    return cpq ? scion_closest_point(dt, (const float*)d_q, n, (scion_cp*)d_r, st, ctr, 0, nullptr)
               : scion_closest_hit(dt, (const scion_ray*)d_q, n, (scion_hit*)d_r, st, ctr, 0, nullptr);
  };
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  std::vector<float> ms;
  for (int i = 0; i < 10; i++) {
    CU(cudaEventRecord(e0));
    CK(run(nullptr, nullptr));
    CU(cudaEventRecord(e1));
    CU(cudaEventSynchronize(e1));
    float t = 0;
    CU(cudaEventElapsedTime(&t, e0, e1));
    if (i) ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  const double mean_ms = (ms[2] + ms[3] + ms[4] + ms[5] + ms[6]) / 5.0;
  // instrumented pass: the reference's cost counters + per-query status
  CK(run(d_st, d_ctr));
  CU(cudaDeviceSynchronize());
  std::vector<scion_counters> ctr(n);
  std::vector<uint32_t> st(n);
  CU(cudaMemcpy(ctr.data(), d_ctr, n * sizeof(scion_counters), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(st.data(), d_st, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  double visits = 0, prims = 0, cold = 0;
  uint64_t errors = 0;
  for (uint64_t i = 0; i < n; i++) {
    visits += ctr[i].node_visits;
    prims += ctr[i].prim_tests;
    cold += ctr[i].cold_loads;
    errors += st[i] != SCION_Q_OK;
  }
  visits /= (double)n; prims /= (double)n; cold /= (double)n;
  // algorithmic bytes per query: hot segment per visit, the rest of the node per cold load
  const double bpq = visits * hot + cold * ((double)li.node_stride - hot) + prims * 36.0 + (cpq ? 32.0 : 40.0);
  std::printf("layout,algorithm,scene,n_gpus,queries,kind,mean_ms,mqueries_per_s,bvh_bytes_per_prim,node_visits,prim_tests,bytes_per_query,achieved_gbs,query_errors,encode\n");
  std::printf("%s,%s,%s,1,%llu,%s,%.4f,%.2f,%.3f,%.2f,%.2f,%.1f,%.1f,%llu,%s\n", layout, cpq ? "cpq" : "chrt", argv[3], (unsigned long long)n, kind.c_str(), mean_ms, (double)n / mean_ms / 1e3,
              (double)node_bytes / (double)nprims, visits, prims, bpq, bpq * (double)n / mean_ms / 1e6, (unsigned long long)errors, host_encode ? "host" : "device");
  cudaFree(d_q); cudaFree(d_r); cudaFree(d_st); cudaFree(d_ctr);
  scion_dtree_free(dt);
  scion_ltree_free(lt);
  scion_scene_free(scene);
  return errors ? 1 : 0;
}
