// Op-count report of a layout's decode (`scionc stats`, the B200 backend's counterpart of the reference CLI's
// `--dump-stats`: "emits op-count JSON"; its DESIGN DECISIONS paragraph: "Interpreter cost counters (loads,
// ALU ops ...) are built into the IR for measuring §7.3-style effects").  Counted on the layout's own expressions, per
// variant arm, with helper functions inlined once per call site:
//   load_slots     stored fields a decode of that variant reads (the reference IR's LoadSlot ops)
//   load_bits      their total width
//   arith / compare / cast / bitcast / call_intrinsic / directed_rounding / select / bit_range / construct
//                  pure-expression ops of the derive / let / key expressions (one count per expression node: a vector
//                  operation counts once, whatever its lane count)
// plus the record geometry (bytes per node, segments) — what the memory-roofline figures are computed from.
#include <functional>
#include <sstream>

#include "layoutc.hpp"

namespace scion::lc {
namespace {

struct Counts {
  uint64_t load_slots = 0, load_bits = 0, arith = 0, compare = 0, cast = 0, bitcast = 0, intrinsic = 0, directed = 0, bit_range = 0, construct = 0, calls_inlined = 0;
  void add(const Counts& o) {
    load_slots += o.load_slots; load_bits += o.load_bits; arith += o.arith; compare += o.compare; cast += o.cast; bitcast += o.bitcast;
    intrinsic += o.intrinsic; directed += o.directed; bit_range += o.bit_range; construct += o.construct; calls_inlined += o.calls_inlined;
  }
  std::string json() const {
    std::ostringstream o;
    o << "{\"load_slots\": " << load_slots << ", \"load_bits\": " << load_bits << ", \"arith\": " << arith << ", \"compare\": " << compare << ", \"cast\": " << cast
      << ", \"bitcast\": " << bitcast << ", \"call_intrinsic\": " << intrinsic << ", \"directed_rounding\": " << directed << ", \"bit_range\": " << bit_range
      << ", \"construct\": " << construct << ", \"calls_inlined\": " << calls_inlined << "}";
    return o.str();
  }
};

struct Counter {
  const Plan& plan;
  const Program& prog;
  explicit Counter(const Plan& p) : plan(p), prog(*p.program) {}
  const Func* func(const std::string& n) const {
    for (auto& f : prog.funcs)
      if (f.name == n) return &f;
    return nullptr;
  }
  void expr(const ExprP& e, Counts& c, uint64_t lanes, int depth) const {
    if (!e) return;
    uint64_t l = lanes;
    switch (e->kind) {
      case Expr::Binary: {
        const std::string& op = e->text;
        if (op == "<" || op == ">" || op == "<=" || op == ">=" || op == "==" || op == "!=") c.compare += l;
        else c.arith += l;
        break;
      }
      case Expr::Unary: c.arith += l; break;
      case Expr::Cast: (e->bitcast ? c.bitcast : c.cast) += 1; break;
      case Expr::Range: c.bit_range += 1; break;
      case Expr::Construct: case Expr::Brace: case Expr::Tuple: c.construct += 1; l = 1; break;
      case Expr::Call: {
        static const std::set<std::string> directed = {"fmul_rd", "fadd_rd", "fsub_rd", "fsub_ru", "fdiv_rd", "frcp_rd"};
        if (directed.count(e->text)) c.directed += l;
        else if (const Func* f = func(e->text)) {
          if (depth < 8) {
            c.calls_inlined += 1;
            body(f->body, c, depth + 1);
          }
        } else c.intrinsic += l;
        break;
      }
      default: break;
    }
    for (auto& a : e->args) expr(a, c, l, depth);
  }
  void body(const std::vector<StmtP>& b, Counts& c, int depth) const {
    for (auto& s : b) {
      expr(s->value, c, 1, depth);
      expr(s->lhs, c, 1, depth);
      expr(s->cond, c, 1, depth);
      body(s->then_body, c, depth);
      body(s->else_body, c, depth);
    }
  }
  // members visible to every variant (outside splits) / inside one arm
  void members(const std::vector<MemberP>& ms, Counts& common, std::map<std::string, Counts>& arms, const std::string& arm) const {
    Counts& c = arm.empty() ? common : arms[arm];
    for (auto& m : ms) {
      switch (m->kind) {
        case MemberNode::Stored:
          for (auto& s : plan.slots)
            if (s.member == m.get()) { c.load_slots += 1; c.load_bits += s.width; }
          break;
        case MemberNode::Derive: case MemberNode::Let: expr(m->value, c, 1, 0); break;
        case MemberNode::Group:
          if (!m->indirect) members(m->members, common, arms, arm);
          break;
        case MemberNode::Split:
          expr(m->value, c, 1, 0);
          for (auto& a : m->arms) {
            const std::string v = arm.empty() ? a.variant : arm;
            expr(a.from_key, arms[v], 1, 0);
            if (a.is_from) {
              std::function<const MemberNode*(const std::vector<MemberP>&)> find = [&](const std::vector<MemberP>& v2) -> const MemberNode* {
                for (auto& g : v2) {
                  if (g->kind == MemberNode::Group && g->indirect && g->group_name == a.from_group) return g.get();
                  if (const MemberNode* r = find(g->members)) return r;
                }
                return nullptr;
              };
              if (const MemberNode* g = find(plan.layout->members)) members(g->members, common, arms, v);
            } else {
              members(a.members, common, arms, v);
            }
          }
          break;
        default: break;
      }
    }
  }
};

}  // namespace

std::string decode_stats_json(const Plan& plan) {
  Counter k(plan);
  Counts common;
  std::map<std::string, Counts> arms;
  for (auto& v : plan.adt->variants) arms[v.name];
  k.members(plan.layout->members, common, arms, "");
  std::ostringstream o;
  o << "{\"layout\": \"" << plan.layout_name << "\", \"family\": " << (int)plan.family << ", \"node_group\": \"" << plan.node_group << "\"";
  if (const Buffer* b = plan.buffer_named(plan.node_group)) {
    o << ", \"node_bytes\": " << b->node_stride() << ", \"segment_bytes\": [";
    for (size_t s = 0; s < b->segments.size(); s++) o << (s ? ", " : "") << b->segments[s].stride_bytes;
    o << "], \"align\": " << b->align;
  }
  o << ", \"stored_fields\": " << plan.slots.size() << ", \"common\": " << common.json() << ", \"variants\": {";
  bool first = true;
  for (auto& v : plan.adt->variants) {
    Counts t = common;
    t.add(arms[v.name]);
    o << (first ? "" : ", ") << "\"" << v.name << "\": {\"arm\": " << arms[v.name].json() << ", \"decode_total\": " << t.json() << "}";
    first = false;
  }
  o << "}}";
  return o.str();
}

}  // namespace scion::lc
