// Scene tools: synthetic scenes and LogicalTree builders.
//
// Stands in for the reference's placeholders src/scene.cpp and src/logical.cpp; the
// contract followed is SPEC.md:523-591 ([MODULE] scene-tools).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "scion_b200.h"

struct scion_scene {
  std::vector<float> tris;  // 9 floats per triangle
  std::string name;
  uint64_t ntris() const { return tris.size() / 9; }
};

struct scion_ltree {
  std::vector<scion_lnode> nodes;   // preorder: left child of i is i+1
  std::vector<float> tris;          // tree order (leaf visit order), 9 floats each
  std::vector<uint32_t> prim_ids;   // tree order -> scene triangle index
  std::vector<float> dop_lo2, dop_hi2;  // 4 per node: min/max of x+y+z, x+y-z, x-y+z, x-y-z
  uint32_t depth = 0;               // root = 0
  // 8-wide collapse (filled by collapse8)
  std::vector<scion_wnode> wnodes;  // preorder
  std::vector<scion_wleaf> wleaves; // DFS slot order
  int32_t wroot = SCION_W_SENTINEL;
  bool has_wide = false;
};

namespace scion {
void make_terrain(uint32_t grid, uint64_t seed, scion_scene& out);
void make_sphere(uint32_t grid, uint64_t seed, scion_scene& out);
void make_cloud(uint64_t npoints, uint64_t seed, scion_scene& out);
void scene_bounds(const scion_scene& s, float lo[3], float hi[3]);

enum class Builder { SAH, Median };
// throws std::runtime_error on bad arguments
void build_binary(const scion_scene& s, Builder kind, uint32_t bins, uint32_t max_leaf, uint32_t max_depth,
                  scion_ltree& out);
void collapse8(scion_ltree& t);
void import_binary(const scion_lnode* nodes, uint64_t nnodes, const float* tris9, uint64_t ntris, scion_ltree& out);
}  // namespace scion
