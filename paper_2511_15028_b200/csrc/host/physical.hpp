// PhysicalTree on the host (buffer id -> byte array; global slot -> scalar;
// root reference; provenance) + the layout registry of the backend.
#pragma once
#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../layoutc/layoutc.hpp"
#include "scene.hpp"

struct scion_ptree {
  std::string layout;                    // registry name
  const scion::lc::Plan* plan = nullptr; // owned by the registry (process lifetime)
  std::vector<std::vector<uint8_t>> buffers;      // indexed by plan buffer id
  std::vector<uint64_t> sizes;                    // byte size per buffer (== buffers[b].size() unless this is a shell, see encode_shell)
  std::vector<uint64_t> counts;                   // element count per buffer (arena: bytes)
  std::vector<std::vector<uint64_t>> seg_bases;   // byte offsets per buffer
  std::vector<std::array<uint8_t, 16>> globals;   // raw little-endian cells, plan.globals order
  uint64_t root0 = 0;
  float carried[6] = {0, 0, 0, 0, 0, 0};
  uint64_t nprims = 0;
};

namespace scion {

struct LayoutEntry {
  std::string name;       // registry name, e.g. "pbrt-q16" (same strings as corpus.cpp:11-25)
  std::string source;     // embedded .scion text
  std::unique_ptr<lc::Program> program;
  std::unique_ptr<lc::Plan> plan;
  bool has_cpq = false;
};

// registry of every layout compiled into the library (parsed + planned lazily, once)
const std::vector<LayoutEntry>& layout_registry();
const LayoutEntry* find_layout(const std::string& name);
// layouts compiled and registered at run time (host/plugin.cpp)
int dyn_layout_count();
const LayoutEntry* dyn_layout_at(int i);
void register_layout_plugin(const std::string& name, const std::string& source, const std::string& work_dir, std::string& log);

// build_physical: throws std::runtime_error (builder hard fault) on capacity violations
void encode_tree(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out);
// device-side encode: sizes, globals, root reference and the per-node job, but no buffer contents
namespace enc { struct EncodeJob; }
void encode_shell(const scion_ltree& t, const LayoutEntry& layout, scion_ptree& out, enc::EncodeJob& job, std::vector<uint32_t>& post);

}  // namespace scion
