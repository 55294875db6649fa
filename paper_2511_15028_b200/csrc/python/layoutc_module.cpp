// _layoutc — Python module of the layout compiler (pybind11), the binding slot of the reference build
// (/root/reference/proj/CMakeLists.txt:74-97 `pybind11_add_module(_layoutc python/layoutc_module.cpp)`; the reference's
// own python/layoutc_module.cpp is a placeholder).  Pure host code: the layout-language front end, the planner and the
// code generators — no CUDA, no device.  The traversal path is reached through the C ABI (include/scion_b200.h), not here.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <string>
#include <vector>

#include "../layoutc/layoutc.hpp"

namespace py = pybind11;
namespace lc = scion::lc;

namespace scion {
struct EmbeddedLayout {
  const char* name;
  const char* source;
};
extern const EmbeddedLayout kEmbeddedLayouts[];
extern const int kEmbeddedLayoutCount;
}  // namespace scion

namespace {
struct Compiled {  // a parsed + planned layout; the Plan points into the Program, so they live together
  std::shared_ptr<lc::Program> program;
  std::shared_ptr<lc::Plan> plan;
};
Compiled compile_text(const std::string& source, const std::string& name) {
  Compiled c;
  c.program = std::make_shared<lc::Program>(lc::parse_program({source}));
  c.plan = std::make_shared<lc::Plan>(lc::plan_layout(*c.program, name));
  return c;
}
Compiled shipped(const std::string& name) {
  for (int i = 0; i < scion::kEmbeddedLayoutCount; i++)
    if (name == scion::kEmbeddedLayouts[i].name) return compile_text(scion::kEmbeddedLayouts[i].source, name);
  throw py::key_error("unknown layout '" + name + "'");
}
}  // namespace

PYBIND11_MODULE(_layoutc, m) {
  m.doc() = "Scion layout compiler for the B200 backend: parse / check / plan / emit (CUDA header, C11 records, op counts)";
  py::register_exception<lc::LayoutError>(m, "LayoutError");
  py::class_<Compiled>(m, "Layout")
      .def_property_readonly("name", [](const Compiled& c) { return c.plan->layout_name; })
      .def_property_readonly("family", [](const Compiled& c) { return (int)c.plan->family; })
      .def_property_readonly("node_group", [](const Compiled& c) { return c.plan->node_group; })
      .def_property_readonly("node_stride", [](const Compiled& c) {
        const lc::Buffer* b = c.plan->buffer_named(c.plan->node_group);
        return b ? b->node_stride() : 0;
      })
      .def_property_readonly("max_leaf", [](const Compiled& c) { return c.plan->max_leaf; })
      .def("plan_json", [](const Compiled& c) { return c.plan->to_json(); }, "MemoryPlan as JSON (buffers, segments, slots @bit offset:width)")
      .def("emit_cuda", [](const Compiled& c) { return lc::emit_cuda(*c.plan); }, "CUDA header: typed node records + decode routines")
      .def("emit_c", [](const Compiled& c) { return lc::emit_c_records(*c.plan); }, "C11 header: typed packed node records + static assertions + slot table")
      .def("stats_json", [](const Compiled& c) { return lc::decode_stats_json(*c.plan); }, "op counts of the decode per variant (--dump-stats)");
  m.def("shipped_layouts", [] {
    std::vector<std::string> v;
    for (int i = 0; i < scion::kEmbeddedLayoutCount; i++) v.push_back(scion::kEmbeddedLayouts[i].name);
    return v;
  }, "registry names of the layouts compiled into the product library");
  m.def("shipped_source", [](const std::string& name) {
    for (int i = 0; i < scion::kEmbeddedLayoutCount; i++)
      if (name == scion::kEmbeddedLayouts[i].name) return std::string(scion::kEmbeddedLayouts[i].source);
    throw py::key_error("unknown layout '" + name + "'");
  });
  m.def("load", &shipped, py::arg("name"), "parse + check + plan a shipped layout");
  m.def("compile", &compile_text, py::arg("source"), py::arg("name") = "user-layout", "parse + check + plan layout-language text; raises LayoutError with the reference's diagnostic class");
}
