// TEST-ONLY: constructors emitted by OUR layout compiler from the REFERENCE's own corpus file (-DGEN_HEADER=..., the
// header is produced at test time by `scionc emit-cuda <layout> /root/reference/proj/corpus/layouts/<file>.scion`) run
// against this library's plan of the same-named layout.  Linked against libscion_b200.so.
#include GEN_HEADER
#include "host/build_ctx.hpp"

namespace {
using LayoutT = scion_gen::GEN_STRUCT;
uint64_t build_root(scion::BuildCtx& b) { return LayoutT::build_node(b, b.view(b.root_id)); }
}  // namespace

extern "C" int ref_build(const scion_ltree* t, scion_ptree** out, char* err, int err_len) {
  static_assert(LayoutT::kHasBuild, "the corpus file carries a build block");
  try {
    const scion::LayoutEntry* e = scion::find_layout(LayoutT::kName);
    if (!e) throw std::runtime_error("unknown layout");
    auto* p = new scion_ptree();
    scion::encode_tree_with(*t, *e, &build_root, *p);
    *out = p;
    return 0;
  } catch (const std::exception& ex) {
    snprintf(err, (size_t)err_len, "%s", ex.what());
    return 1;
  }
}
