// TEST INFRASTRUCTURE — not part of the product.
// Driver (our own code) that links against the reference's real front-end TUs,
// compiled in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/.  It runs the reference's own pipeline
//   parse_corpus -> layout_adt -> check_layout -> plan_layout
// (idiom of /root/reference/proj/tests/test_plan.cpp:40-57) and dumps every
// buffer / segment / slot as JSON, so that our planner (product) and the
// oracle's slot tables can be pinned against the reference planner
// (/root/reference/proj/src/plan.cpp:349).
//
// usage: ref_probe <corpus-layout-name | /abs/path/layout.scion [/abs/extra.scion ...]> ...
#include <algorithm>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "layoutc/corpus.hpp"
#include "layoutc/plan.hpp"
#include "layoutc/sema.hpp"

using namespace layoutc;

static std::string esc(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

static bool dump_one(const std::string& label, const std::vector<std::string>& files, std::ostream& os) {
  SourceSet ss;
  ParseResult r = parse_corpus(files, &ss);
  if (!r.ok()) {
    std::cerr << label << ": parse failed\n";
    return false;
  }
  Program program = std::move(r.program);
  LayoutSpec* layout = nullptr;
  for (auto& l : program.layouts)
    if (program.find_build(l.name)) layout = &l;
  if (!layout && !program.layouts.empty()) layout = &program.layouts.back();
  if (!layout) return false;
  const AdtDecl* adt = layout_adt(program, *layout);
  if (!adt) return false;
  auto diags = check_layout(*adt, *layout, program);
  if (!diags.empty()) {
    std::cerr << label << ": check_layout diagnostics: " << diags.size() << "\n";
    return false;
  }
  // the reference's own check_build (src/sema_build.cpp) over the file's build block, when it carries one
  if (const BuildSpec* cb = program.find_build(layout->name)) {
    auto bd = check_build(*adt, *layout, const_cast<BuildSpec&>(*cb), program);
    if (!bd.empty()) {
      std::cerr << label << ": check_build diagnostics: " << bd.size() << "\n";
      for (auto& d : bd) std::cerr << "  " << d.message << "\n";
      return false;
    }
    std::cerr << label << ": check_build ok\n";
  }
  MemoryPlan plan = plan_layout(*adt, *layout, program);
  os << "  \"" << esc(label) << "\": {\n";
  os << "    \"adt\": \"" << esc(plan.adt_name) << "\",\n    \"ref\": [";
  for (size_t i = 0; i < plan.components.size(); i++) {
    if (i) os << ", ";
    os << "{\"name\": \"" << esc(plan.components[i].name) << "\", \"type\": \""
       << esc(type_to_string(*plan.components[i].type)) << "\"}";
  }
  os << "],\n    \"globals\": [";
  for (size_t i = 0; i < plan.globals.size(); i++) {
    if (i) os << ", ";
    os << "{\"name\": \"" << esc(plan.globals[i].name) << "\", \"type\": \""
       << esc(type_to_string(*plan.globals[i].type)) << "\", \"inferred\": "
       << (plan.globals[i].inferred ? "true" : "false") << "}";
  }
  os << "],\n    \"buffers\": [\n";
  for (size_t b = 0; b < plan.buffers.size(); b++) {
    const BufferDesc& bd = plan.buffers[b];
    os << "      {\"id\": " << bd.id << ", \"name\": \"" << esc(bd.name) << "\", \"arena\": "
       << (bd.is_arena ? "true" : "false") << ", \"global_array\": "
       << (bd.is_global_array ? "true" : "false") << ", \"align\": " << bd.align_bytes
       << ", \"count\": \"" << esc(bd.count_name) << "\", \"node_stride\": " << node_stride_bytes(bd)
       << ", \"segments\": [";
    for (size_t s = 0; s < bd.segments.size(); s++) {
      if (s) os << ", ";
      os << "{\"stride_bits\": " << bd.segments[s].stride_bits << ", \"stride_bytes\": "
         << bd.segments[s].stride_bytes << ", \"tile\": " << bd.segments[s].tile << "}";
    }
    os << "]}" << (b + 1 < plan.buffers.size() ? "," : "") << "\n";
  }
  os << "    ],\n    \"slots\": [\n";
  // deterministic order: by (buffer, segment, offset, name)
  std::vector<const FieldSlot*> slots;
  for (auto& kv : plan.slots) slots.push_back(&kv.second);
  std::sort(slots.begin(), slots.end(), [](const FieldSlot* a, const FieldSlot* b) {
    if (a->buffer != b->buffer) return a->buffer < b->buffer;
    if (a->segment != b->segment) return a->segment < b->segment;
    if (a->offset != b->offset) return a->offset < b->offset;
    return a->name < b->name;
  });
  for (size_t i = 0; i < slots.size(); i++) {
    const FieldSlot& s = *slots[i];
    os << "      {\"name\": \"" << esc(s.name) << "\", \"buffer\": " << s.buffer << ", \"segment\": "
       << s.segment << ", \"offset\": " << s.offset << ", \"width\": " << s.width << ", \"type\": \""
       << esc(s.type ? type_to_string(*s.type) : "") << "\"}" << (i + 1 < slots.size() ? "," : "") << "\n";
  }
  os << "    ],\n    \"variant_home\": {";
  bool first = true;
  for (auto& kv : plan.variant_home) {
    if (!first) os << ", ";
    first = false;
    os << "\"" << esc(kv.first) << "\": " << kv.second;
  }
  os << "}\n  }";
  return true;
}

int main(int argc, char** argv) {
  std::ostringstream os;
  os << "{\n";
  bool first = true;
  int rc = 0;
  std::vector<std::string> names;
  for (int i = 1; i < argc; i++) names.push_back(argv[i]);
  if (names.empty())
    for (auto& l : corpus_layouts()) names.push_back(l.name);
  for (auto& n : names) {
    std::vector<std::string> files;
    std::string label = n;
    if (!n.empty() && n[0] == '/') {
      files = {"lib/geometry.scion", n};
      size_t slash = n.find_last_of('/');
      label = n.substr(slash + 1);
      size_t dot = label.find_last_of('.');
      if (dot != std::string::npos) label = label.substr(0, dot);
    } else {
      files = corpus_files_for_layout(n);
    }
    std::ostringstream one;
    try {
      if (dump_one(label, files, one)) {
        if (!first) os << ",\n";
        first = false;
        os << one.str();
      } else {
        rc = 1;
      }
    } catch (const std::exception& e) {
      std::cerr << n << ": " << e.what() << "\n";
      rc = 1;
    }
  }
  os << "\n}\n";
  std::cout << os.str();
  return rc;
}
