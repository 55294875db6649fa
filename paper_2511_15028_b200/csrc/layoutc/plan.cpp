// Memory planner: layout AST -> buffers / segments / bit-exact slots.
//
// The packing rules are the reference planner's (/root/reference/proj/src/plan.cpp):
//   * fields packed tightly in declaration order, no implicit padding        (:81-97)
//   * explicit numeric members add padding bits                              (:98-100)
//   * every split arm overlays the same region; its width is the widest arm  (:126-141)
//   * `---` closes a segment; each segment's stride is rounded up to whole
//     bytes and to the group's `align`                                       (:44-63, :103-107)
//   * segment s starts at round_up(sum of earlier segments' count*stride, align) (:333-347)
//   * a top-level `T[len]` field is a global array buffer of stride ceil(bits/8) (:195-210)
//   * a direct group indexed by a `ptr` reference component is an arena whose
//     elements are addressed by byte offset                                  (:150-155, :315-318)
//   * tree-carried reference components get `__ref_<name>` globals           (:233-241)
// tests/test_layoutc.py pins this planner against the reference planner's own output
// (tests/golden/ref_plans.json, produced by oracle/ref_probe.cpp) slot by slot.
#include <algorithm>
#include <functional>
#include <sstream>

#include "layoutc.hpp"

namespace scion::lc {

static uint64_t round_up(uint64_t v, uint64_t a) { return a <= 1 ? v : (v + a - 1) / a * a; }

uint64_t Buffer::bytes(uint64_t count, std::vector<uint64_t>* bases) const {
  uint64_t base = 0;
  if (bases) bases->clear();
  for (auto& s : segments) {
    base = round_up(base, align);
    if (bases) bases->push_back(base);
    base += count * s.stride_bytes;
  }
  return base;
}

uint64_t Plan::type_bits(const TypeP& t) const {
  switch (t->kind) {
    case Type::Int: case Type::Float: return t->width;
    case Type::Bool: return 1;
    case Type::Ptr: return 64;
    case Type::Vec: return type_bits(t->elem) * t->lanes;
    case Type::Array:
      if (!t->len_field.empty()) throw LayoutError("dynamically sized arrays may only appear at the layout top level");
      return type_bits(t->elem) * t->lanes;
    case Type::Tuple: {
      uint64_t w = 0;
      for (auto& m : t->members) w += type_bits(m);
      return w;
    }
    case Type::Named: {
      const TypeDecl* d = program->find_type(t->name);
      if (!d) throw LayoutError("unknown type '" + t->name + "'");
      if (d->is_adt()) throw LayoutError("ADT '" + t->name + "' cannot be stored by value");
      uint64_t w = 0;
      for (auto& f : d->fields) w += type_bits(f.type);
      return w;
    }
  }
  return 0;
}

namespace {

struct Planner {
  Plan& plan;
  const Layout& layout;

  struct Cursor {
    int buf = -1;
    uint64_t bit = 0;
    int segment = 0;
  };

  void close_segment(Cursor& c) {
    Buffer& b = plan.buffers[(size_t)c.buf];
    Segment s;
    s.stride_bits = c.bit;
    s.stride_bytes = round_up((c.bit + 7) / 8, b.align);
    b.segments.push_back(s);
    c.bit = 0;
    c.segment++;
  }

  void lay(const MemberNode& m, Cursor& c) {
    switch (m.kind) {
      case MemberNode::Stored: {
        Slot s;
        s.name = m.name;
        s.buffer = c.buf;
        s.segment = c.segment;
        s.offset = c.bit;
        s.width = (uint32_t)plan.type_bits(m.type);
        if (s.width == 0) throw LayoutError("zero-width field '" + m.name + "'");
        s.type = m.type;
        s.member = &m;
        plan.slots.push_back(s);
        c.bit += s.width;
        break;
      }
      case MemberNode::Padding: c.bit += m.padding_bits; break;
      case MemberNode::Derive: case MemberNode::Let: break;
      case MemberNode::Separator:
        if (plan.buffers[(size_t)c.buf].is_arena) throw LayoutError("--- is not supported in address-referenced groups");
        close_segment(c);
        break;
      case MemberNode::Group:
        if (m.indirect) { plan_group(m); break; }
        throw LayoutError("nested direct (tiled) groups are not supported by the B200 backend");
      case MemberNode::Split: {
        uint64_t base = c.bit, widest = 0;
        int seg0 = c.segment;
        for (auto& arm : m.arms) {
          if (arm.is_from) continue;
          c.bit = base;
          for (auto& am : arm.members) lay(*am, c);
          if (c.segment != seg0) throw LayoutError("segment boundaries inside split arms are not supported");
          widest = std::max(widest, c.bit - base);
        }
        c.bit = base + widest;
        break;
      }
    }
  }

  void plan_group(const MemberNode& g) {
    Buffer b;
    b.id = (int)plan.buffers.size();
    b.name = g.group_name.empty() ? "group" + std::to_string(b.id) : g.group_name;
    b.align = g.align ? (uint32_t)g.align : 1;
    if (!g.indirect && !g.index_binding.empty())
      for (auto& r : layout.ref)
        if (r.name == g.index_binding && r.type->kind == Type::Ptr) b.is_arena = true;
    if (g.size_expr && g.size_expr->kind == Expr::Ident) b.count_name = g.size_expr->text;
    else b.count_name = "__count_" + b.name;
    plan.buffers.push_back(b);
    Cursor c;
    c.buf = b.id;
    for (auto& m : g.members) lay(*m, c);
    close_segment(c);
    auto& segs = plan.buffers[(size_t)b.id].segments;
    while (!segs.empty() && segs.back().stride_bits == 0) segs.pop_back();
  }

  // which buffer materialises `variant` (plan.cpp:245-303): a `from` arm homes in the
  // indirect group, an inline arm in the enclosing direct group if it owns storage
  int find_home(const std::string& variant) {
    int home = -1;
    std::function<void(const std::vector<MemberP>&, int)> walk = [&](const std::vector<MemberP>& ms, int enclosing) {
      for (auto& m : ms) {
        if (m->kind == MemberNode::Group) {
          if (m->indirect) continue;
          const Buffer* b = plan.buffer_named(m->group_name.empty() ? "" : m->group_name);
          int id = -1;
          for (auto& bb : plan.buffers)
            if (group_of.count(bb.id) && group_of[bb.id] == m.get()) id = bb.id;
          (void)b;
          walk(m->members, id);
        } else if (m->kind == MemberNode::Split) {
          for (auto& arm : m->arms) {
            if (arm.variant == variant) {
              if (arm.is_from) {
                const Buffer* ib = plan.buffer_named(arm.from_group);
                home = ib ? ib->id : -1;
              } else {
                home = (enclosing >= 0 && !plan.buffers[(size_t)enclosing].segments.empty()) ? enclosing : -1;
              }
            }
            walk(arm.members, enclosing);
          }
        }
      }
    };
    walk(layout.members, -1);
    return home;
  }
  std::map<int, const MemberNode*> group_of;

  void run() {
    plan.ref = layout.ref;
    // names of globals that are element counts (filled by the builder's count pass)
    std::set<std::string> counts;
    std::function<void(const std::vector<MemberP>&)> scan = [&](const std::vector<MemberP>& ms) {
      for (auto& m : ms) {
        if (m->kind == MemberNode::Stored && m->type->kind == Type::Array && !m->type->len_field.empty()) counts.insert(m->type->len_field);
        if (m->kind == MemberNode::Group) {
          if (m->size_expr && m->size_expr->kind == Expr::Ident) counts.insert(m->size_expr->text);
          scan(m->members);
        }
      }
    };
    scan(layout.members);
    for (auto& m : layout.members) {
      switch (m->kind) {
        case MemberNode::Stored:
          if (m->type->kind == Type::Array && !m->type->len_field.empty()) {
            Buffer b;
            b.id = (int)plan.buffers.size();
            b.name = m->name;
            b.is_global_array = true;
            b.elem_type = m->type->elem;
            b.count_name = m->type->len_field;
            Segment s;
            s.stride_bits = plan.type_bits(m->type->elem);
            s.stride_bytes = (s.stride_bits + 7) / 8;
            b.segments.push_back(s);
            plan.buffers.push_back(b);
          } else {
            plan.globals.push_back({m->name, m->type, counts.count(m->name) > 0});
          }
          break;
        case MemberNode::Group: {
          size_t before = plan.buffers.size();
          plan_group(*m);
          // the group's own buffer is the first one pushed by plan_group
          group_of[(int)before] = m.get();
          break;
        }
        case MemberNode::Split: throw LayoutError("top-level splits are not supported");
        case MemberNode::Separator: throw LayoutError("--- outside a group");
        default: break;
      }
    }
    for (size_t i = 1; i < layout.ref.size(); i++) plan.globals.push_back({"__ref_" + layout.ref[i].name, layout.ref[i].type, false});
    for (auto& v : plan.adt->variants) plan.variant_home[v.name] = find_home(v.name);
  }
};

void json_str(std::ostringstream& os, const std::string& s) {
  os << '"';
  for (char c : s) {
    if (c == '"' || c == '\\') os << '\\';
    os << c;
  }
  os << '"';
}

}  // namespace

std::string ident_of(const std::string& n) {
  std::string o;
  for (char c : n) o += (isalnum((unsigned char)c) ? c : '_');
  return o;
}

Plan plan_layout(const Program& program, const std::string& registry_name) {
  if (program.layouts.empty()) throw LayoutError("no layout declaration found");
  const Layout& layout = program.layouts.back();
  Plan plan;
  plan.layout_name = registry_name;
  plan.program = &program;
  plan.layout = &layout;
  plan.adt = program.find_type(layout.name);
  if (!plan.adt || !plan.adt->is_adt()) throw LayoutError("layout '" + layout.name + "' does not name an ADT");
  check_layout(program, layout, *plan.adt);
  plan.build_order = program.build_orders.empty() ? "pre" : program.build_orders.back();
  Planner p{plan, layout};
  p.run();

  // family from the ADT's shape (corpus.hpp:11 Family)
  auto has_field = [&](const std::vector<Param>& fs, const char* n) {
    for (auto& f : fs)
      if (f.name == n) return true;
    return false;
  };
  const Variant* interior = nullptr;
  const Variant* leaf = nullptr;
  for (auto& v : plan.adt->variants) {
    if (v.name == "Interior") interior = &v;
    if (v.name == "Leaf") leaf = &v;
  }
  if (!interior || !leaf) throw LayoutError("the B200 backend needs Interior and Leaf variants");
  if (has_field(interior->fields, "children")) plan.family = Family::Bvh8;
  else if (has_field(plan.adt->fields, "lo2")) plan.family = Family::Dop14;
  else plan.family = Family::Bvh2;
  for (auto& f : leaf->fields)
    if (f.name == "nprims" && f.type->kind == Type::Int) plan.max_leaf = f.type->width >= 32 ? 0xFFFFFFFFu : ((1u << f.type->width) - 1);
  if (plan.family == Family::Bvh8) {
    // 8-wide leaves are bit-stolen into the reference: nprims-1 occupies bits [2:6] -> <= 32
    plan.max_leaf = std::min<uint32_t>(plan.max_leaf, 32);
  }
  // the node group: the Interior variant's home buffer
  int home = plan.variant_home.count("Interior") ? plan.variant_home["Interior"] : -1;
  if (home >= 0) plan.node_group = plan.buffers[(size_t)home].name;
  return plan;
}

std::string Plan::to_json() const {
  std::ostringstream os;
  os << "{\"layout\": ";
  json_str(os, layout_name);
  os << ", \"adt\": ";
  json_str(os, adt->name);
  os << ", \"family\": " << (int)family << ", \"build_order\": ";
  json_str(os, build_order);
  os << ", \"max_leaf\": " << max_leaf << ", \"node_group\": ";
  json_str(os, node_group);
  os << ", \"ref\": [";
  for (size_t i = 0; i < ref.size(); i++) {
    os << (i ? ", " : "") << "{\"name\": ";
    json_str(os, ref[i].name);
    os << ", \"type\": ";
    json_str(os, ref[i].type->str());
    os << "}";
  }
  os << "], \"globals\": [";
  for (size_t i = 0; i < globals.size(); i++) {
    os << (i ? ", " : "") << "{\"name\": ";
    json_str(os, globals[i].name);
    os << ", \"type\": ";
    json_str(os, globals[i].type->str());
    os << ", \"inferred\": " << (globals[i].inferred ? "true" : "false") << "}";
  }
  os << "], \"buffers\": [";
  for (size_t i = 0; i < buffers.size(); i++) {
    const Buffer& b = buffers[i];
    os << (i ? ", " : "") << "{\"id\": " << b.id << ", \"name\": ";
    json_str(os, b.name);
    os << ", \"arena\": " << (b.is_arena ? "true" : "false") << ", \"global_array\": " << (b.is_global_array ? "true" : "false")
       << ", \"align\": " << b.align << ", \"count\": ";
    json_str(os, b.count_name);
    os << ", \"node_stride\": " << b.node_stride() << ", \"segments\": [";
    for (size_t s = 0; s < b.segments.size(); s++)
      os << (s ? ", " : "") << "{\"stride_bits\": " << b.segments[s].stride_bits << ", \"stride_bytes\": " << b.segments[s].stride_bytes << "}";
    os << "]}";
  }
  os << "], \"slots\": [";
  std::vector<const Slot*> ss;
  for (auto& s : slots) ss.push_back(&s);
  std::stable_sort(ss.begin(), ss.end(), [](const Slot* a, const Slot* b) {
    if (a->buffer != b->buffer) return a->buffer < b->buffer;
    if (a->segment != b->segment) return a->segment < b->segment;
    if (a->offset != b->offset) return a->offset < b->offset;
    return a->name < b->name;
  });
  for (size_t i = 0; i < ss.size(); i++) {
    os << (i ? ", " : "") << "{\"name\": ";
    json_str(os, ss[i]->name);
    os << ", \"buffer\": " << ss[i]->buffer << ", \"segment\": " << ss[i]->segment << ", \"offset\": " << ss[i]->offset
       << ", \"width\": " << ss[i]->width << ", \"type\": ";
    json_str(os, ss[i]->type->str());
    os << "}";
  }
  os << "], \"variant_home\": {";
  bool first = true;
  for (auto& kv : variant_home) {
    if (!first) os << ", ";
    first = false;
    json_str(os, kv.first);
    os << ": " << kv.second;
  }
  os << "}}";
  return os.str();
}

}  // namespace scion::lc
