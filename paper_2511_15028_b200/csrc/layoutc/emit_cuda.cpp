// emit_cuda — CUDA codegen backend of the layout compiler.
//
// Fills, for CUDA, the slot the reference reserves for emit_c ("packed record
// declarations matching MemoryPlan strides bit-for-bit ... a static assertion on node size ...
// deterministic output (golden-testable)").  Per layout it emits one header with
//   * the device node record(s) (one per segment) + static_asserts against the planned stride,
//   * slot offset/width constants,
//   * the record types and helper `func`s the layout's derive expressions reach,
//   * `decode()` — reference + tree view -> ADT view (variant, bounds, children | prim range),
//     i.e. destructor specialisation (Alg. 1 / src/specialize.cpp:20-122) resolved at compile
//     time into constant-offset extractions, and `decode_cold()` for the fields that live
//     behind a `---` separator.
// The DSL is C-like; expressions translate 1:1 (as -> scion::as_*, to -> bit casts,
// x[a:b] -> scion::bits<a,b>, fmul_rd -> __fmul_rd ...) and C++ overload resolution against
// device/scion_rt.cuh does the typing.  The traversal kernels (device/traverse.cuh) are
// templates over the emitted struct.
#include <algorithm>
#include <functional>
#include <numeric>
#include <sstream>

#include "layoutc.hpp"

namespace scion::lc {
namespace {

struct Emitter {
  const Plan& plan;
  const Program& prog;
  std::ostringstream out;
  std::string ref_ctype;
  bool ref_is_struct = false;
  std::set<std::string> global_names, array_names, ref_names;
  std::set<std::string> used_funcs;  // reachable helper funcs
  std::vector<std::string> func_order;

  explicit Emitter(const Plan& p) : plan(p), prog(*p.program) {}

  // ------------------------------------------------------------------ types
  std::string ctype(const TypeP& t) const {
    switch (t->kind) {
      case Type::Int: return t->width <= 32 ? (t->is_signed ? "int32_t" : "uint32_t") : (t->is_signed ? "int64_t" : "uint64_t");
      case Type::Float: return "float";
      case Type::Bool: return "bool";
      case Type::Ptr: return "uint64_t";
      case Type::Vec: return "scion::vec<" + ctype(t->elem) + ", " + std::to_string(t->lanes) + ">";
      case Type::Array:
        if (!t->len_field.empty()) return "scion::Slice";
        return "scion::vec<" + ctype(t->elem) + ", " + std::to_string(t->lanes) + ">";
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        if (d && d->is_adt()) return "Ref";
        return "rec_" + t->name;
      }
      case Type::Tuple: return "Ref";
    }
    return "void";
  }

  // ------------------------------------------------------------------ expressions
  static bool is_intrinsic(const std::string& n) {
    static const std::set<std::string> s = {"dot", "cross", "cross_", "select", "min", "max", "floorf", "ceilf", "abs", "sum", "all",
                                            "fmul_rd", "fadd_rd", "fsub_rd", "fsub_ru", "fdiv_rd", "frcp_rd"};
    return s.count(n) > 0;
  }
  std::string float_lit(const std::string& s) const {
    std::string t = s;
    if (t.find('.') == std::string::npos && t.find('e') == std::string::npos && t.find('E') == std::string::npos) t += ".0";
    return t + "f";
  }
  // `in_layout`: identifiers may name reference components / globals
  std::string ex(const ExprP& e, bool in_layout) {
    switch (e->kind) {
      case Expr::IntLit: {
        std::string s = std::to_string(e->ival);
        if (e->ival > 0x7fffffffull) return s + (e->ival > 0xffffffffull ? "ull" : "u");
        return e->has_u ? s + "u" : s;
      }
      case Expr::FloatLit: return float_lit(e->text);
      case Expr::BuildChild:  // constructor context: build the child, the value is its reference
        return "(uint64_t)b__.template child<Self__>(n__." + e->text + ")";
      case Expr::Ident:
        if (e->text == "inf") return "scion::inf()";
        if (in_build && e->text == "this") return "this__";
        if (in_layout && ref_names.count(e->text)) return ref_is_struct ? "ref__." + e->text : "ref__";
        return e->text;
      case Expr::Binary: return "(" + ex(e->args[0], in_layout) + " " + e->text + " " + ex(e->args[1], in_layout) + ")";
      case Expr::Unary: return "(" + e->text + ex(e->args[0], in_layout) + ")";
      case Expr::Call: {
        std::string fn;
        if (in_build && e->text == "append") {  // append(data, n): copy the leaf's primitives behind the cursor, the value is the start
          if (e->args.size() != 2) throw LayoutError("append takes (data, count)");
          return "b__.append(n__." + ex(e->args[0], in_layout) + ", (uint64_t)(" + ex(e->args[1], in_layout) + "))";
        }
        if (is_intrinsic(e->text)) {
          fn = e->text == "cross_" ? "cross" : e->text == "floorf" ? "floorf_" : e->text == "ceilf" ? "ceilf_" : e->text;
          fn = "scion::" + fn;
        } else {
          fn = "fn_" + e->text;
        }
        std::string s = fn + "(";
        for (size_t i = 0; i < e->args.size(); i++) s += (i ? ", " : "") + ex(e->args[i], in_layout);
        return s + ")";
      }
      case Expr::Member:
        if (in_layout && e->args[0]->kind == Expr::Ident && e->args[0]->text == "parent") return "ref__." + e->text;
        return ex(e->args[0], in_layout) + "." + e->text;
      case Expr::Index: {
        // constant lane index -> operator[]; dynamic lane index -> scion::get_lane
        if (e->args[1]->kind == Expr::IntLit) return ex(e->args[0], in_layout) + "[" + std::to_string(e->args[1]->ival) + "]";
        return "scion::get_lane(" + ex(e->args[0], in_layout) + ", " + ex(e->args[1], in_layout) + ")";
      }
      case Expr::Range: {
        const ExprP& base = e->args[0];
        if (in_layout && base->kind == Expr::Ident && array_names.count(base->text))
          return "scion::make_slice((uint64_t)(" + ex(e->args[1], in_layout) + "), (uint64_t)(" + ex(e->args[2], in_layout) + "))";
        if (e->args[1]->kind != Expr::IntLit || e->args[2]->kind != Expr::IntLit) throw LayoutError("bit ranges need literal bounds");
        return "scion::bits<" + std::to_string(e->args[1]->ival) + ", " + std::to_string(e->args[2]->ival) + ">(" + ex(base, in_layout) + ")";
      }
      case Expr::Cast: {
        std::string a = ex(e->args[0], in_layout);
        const TypeP& t = e->type;
        const Type* leaf = t.get();
        while (leaf->kind == Type::Vec) leaf = leaf->elem.get();
        if (e->bitcast) {
          if (t->kind == Type::Float) return "scion::bit_to_f32(" + a + ")";
          if (t->kind == Type::Int && t->width == 32) return std::string(t->is_signed ? "scion::bit_to_i32(" : "scion::bit_to_u32(") + a + ")";
          throw LayoutError("unsupported bit cast target " + t->str());
        }
        if (leaf->kind == Type::Float) return "scion::as_<" + ctype(t) + ">(" + a + ")";
        if (leaf->kind == Type::Int) {
          if (leaf->is_signed) return "scion::as_sint<" + std::to_string(leaf->width) + ">(" + a + ")";
          if (leaf->width > 32) return "scion::as_uint64<" + std::to_string(leaf->width) + ">(" + a + ")";
          return "scion::as_uint<" + std::to_string(leaf->width) + ">(" + a + ")";
        }
        if (leaf->kind == Type::Ptr) return "(uint64_t)(" + a + ")";
        throw LayoutError("unsupported cast target " + t->str());
      }
      case Expr::Construct: case Expr::Brace: case Expr::Tuple: {
        std::string s = e->kind == Expr::Construct ? ctype(e->type) : e->kind == Expr::Tuple ? std::string("Ref") : std::string();
        s += "{";
        for (size_t i = 0; i < e->args.size(); i++) s += (i ? ", " : "") + ex(e->args[i], in_layout);
        return s + "}";
      }
    }
    return "?";
  }

  void collect_calls(const ExprP& e, std::vector<std::string>& calls) const {
    if (!e) return;
    if (e->kind == Expr::Call && !is_intrinsic(e->text)) calls.push_back(e->text);
    for (auto& a : e->args) collect_calls(a, calls);
  }
  void collect_calls(const std::vector<StmtP>& body, std::vector<std::string>& calls) const {
    for (auto& s : body) {
      collect_calls(s->value, calls);
      collect_calls(s->lhs, calls);
      collect_calls(s->cond, calls);
      collect_calls(s->then_body, calls);
      collect_calls(s->else_body, calls);
    }
  }
  void collect_idents(const ExprP& e, std::set<std::string>& ids) const {
    if (!e) return;
    if (e->kind == Expr::Ident) ids.insert(e->text);
    for (auto& a : e->args) collect_idents(a, ids);
  }
  const Func* find_func(const std::string& n) const {
    for (auto& f : prog.funcs)
      if (f.name == n) return &f;
    return nullptr;
  }
  void reach(const std::string& fn) {
    if (used_funcs.count(fn)) return;
    const Func* f = find_func(fn);
    if (!f) throw LayoutError("call to unknown function '" + fn + "'");
    used_funcs.insert(fn);
    std::vector<std::string> calls;
    collect_calls(f->body, calls);
    for (auto& c : calls) reach(c);
    func_order.push_back(fn);  // callees first
  }
  void reach_members(const std::vector<MemberP>& ms) {
    for (auto& m : ms) {
      std::vector<std::string> calls;
      collect_calls(m->value, calls);
      collect_calls(m->size_expr, calls);
      for (auto& c : calls) reach(c);
      reach_members(m->members);
      for (auto& a : m->arms) {
        std::vector<std::string> k;
        collect_calls(a.from_key, k);
        for (auto& c : k) reach(c);
        reach_members(a.members);
      }
    }
  }

  // ------------------------------------------------------------------ function bodies
  void emit_stmts(const std::vector<StmtP>& body, int ind) {
    std::string pad((size_t)ind * 2, ' ');
    for (auto& s : body) {
      switch (s->kind) {
        case Stmt::Let:
          out << pad << (s->is_mut ? "" : "const ") << ctype(s->type) << " " << s->name << " = " << ex(s->value, false) << ";\n";
          break;
        case Stmt::Assign:
          if (s->lhs->kind == Expr::Index && s->lhs->args[1]->kind != Expr::IntLit)
            out << pad << "scion::set_lane(" << ex(s->lhs->args[0], false) << ", " << ex(s->lhs->args[1], false) << ", " << ex(s->value, false) << ");\n";
          else
            out << pad << ex(s->lhs, false) << " = " << ex(s->value, false) << ";\n";
          break;
        case Stmt::If:
          out << pad << "if (" << ex(s->cond, false) << ") {\n";
          emit_stmts(s->then_body, ind + 1);
          if (!s->else_body.empty()) {
            out << pad << "} else {\n";
            emit_stmts(s->else_body, ind + 1);
          }
          out << pad << "}\n";
          break;
        case Stmt::Return:
          if (s->value && (s->value->kind == Expr::Brace)) out << pad << "return " << cur_ret << ex(s->value, false) << ";\n";
          else out << pad << "return " << (s->value ? ex(s->value, false) : "") << ";\n";
          break;
        case Stmt::ExprS: out << pad << ex(s->value, false) << ";\n"; break;
      }
    }
  }
  std::string cur_ret;
  bool in_build = false;  // emitting a constructor of the build block: `this`, `append`, `build child` are legal

  // ------------------------------------------------------------------ field extraction
  std::string extract(const TypeP& t, uint64_t off, const std::string& words) const {
    auto o = std::to_string(off);
    switch (t->kind) {
      case Type::Float: return "scion::extf<" + o + ">(" + words + ")";
      case Type::Bool: return "(scion::ext32<" + o + ", 1>(" + words + ") != 0u)";
      case Type::Ptr: return "scion::ext64<" + o + ", 64>(" + words + ")";
      case Type::Int: {
        std::string w = std::to_string(t->width);
        if (t->width > 32) return "scion::ext64<" + o + ", " + w + ">(" + words + ")";
        std::string u = "scion::ext32<" + o + ", " + w + ">(" + words + ")";
        return t->is_signed ? "scion::as_sint<" + w + ">(" + u + ")" : u;
      }
      case Type::Vec: case Type::Array: {
        uint64_t ew = plan.type_bits(t->elem);
        std::string s = ctype(t) + "{";
        for (uint32_t i = 0; i < t->lanes; i++) s += (i ? ", " : "") + extract(t->elem, off + i * ew, words);
        return s + "}";
      }
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        std::string s = ctype(t) + "{";
        uint64_t o2 = off;
        for (size_t i = 0; i < d->fields.size(); i++) {
          s += (i ? ", " : "") + extract(d->fields[i].type, o2, words);
          o2 += plan.type_bits(d->fields[i].type);
        }
        return s + "}";
      }
      case Type::Tuple: break;
    }
    throw LayoutError("cannot load a value of type " + t->str());
  }

  // typed store of `val` at bit offset `off` of the staged record image `words` (the inverse of extract)
  void deposit(const TypeP& t, uint64_t off, const std::string& words, const std::string& val, const std::string& pad) {
    auto o = std::to_string(off);
    switch (t->kind) {
      case Type::Float: out << pad << "scion::dep32<" << o << ", 32>(" << words << ", scion::f2u(" << val << "));\n"; return;
      case Type::Bool: out << pad << "scion::dep32<" << o << ", 1>(" << words << ", (" << val << ") ? 1u : 0u);\n"; return;
      case Type::Ptr: out << pad << "scion::dep64<" << o << ", 64>(" << words << ", (uint64_t)(" << val << "));\n"; return;
      case Type::Int:
        if (t->width > 32) out << pad << "scion::dep64<" << o << ", " << t->width << ">(" << words << ", (uint64_t)(" << val << "));\n";
        else out << pad << "scion::dep32<" << o << ", " << t->width << ">(" << words << ", (uint32_t)(" << val << "));\n";
        return;
      case Type::Vec: case Type::Array: {
        if (!t->len_field.empty()) break;
        uint64_t ew = plan.type_bits(t->elem);
        for (uint32_t i = 0; i < t->lanes; i++) deposit(t->elem, off + i * ew, words, val + "[" + std::to_string(i) + "]", pad);
        return;
      }
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        if (!d || d->is_adt()) break;
        uint64_t o2 = off;
        for (auto& f : d->fields) {
          deposit(f.type, o2, words, val + "." + f.name, pad);
          o2 += plan.type_bits(f.type);
        }
        return;
      }
      case Type::Tuple: break;
    }
    throw LayoutError("cannot store a value of type " + t->str());
  }

  // ------------------------------------------------------------------ constructor emission (build blocks)
  // SPEC.md:276-284 specialize_constructors / PAPER.md:1495-1569: per variant one function that reserves this node's
  // storage (before the children for order=pre, after them for order=post), evaluates the build statements — typed stores
  // into a staged image of the record, `append` cursors, recursive child builds through the build context B
  // (host/build_ctx.hpp) — and returns the node's reference.
  bool is_child_type(const TypeP& t) const {
    const Type* u = t.get();
    if ((u->kind == Type::Array || u->kind == Type::Vec) && u->len_field.empty()) u = u->elem.get();
    if (u->kind != Type::Named) return false;
    const TypeDecl* d = prog.find_type(u->name);
    return d && d->is_adt();
  }
  bool stmt_builds_child(const StmtP& st, const BuildCtor& c) const {
    std::function<bool(const ExprP&)> has = [&](const ExprP& e) -> bool {
      if (!e) return false;
      if (e->kind == Expr::BuildChild) return true;
      for (auto& a : e->args)
        if (has(a)) return true;
      return false;
    };
    if (has(st->value) || has(st->lhs) || has(st->cond)) return true;
    if (st->kind == Stmt::Build && !st->value)
      for (auto& pa : c.params)
        if (pa.name == st->name && is_child_type(pa.type)) return true;
    return false;
  }
  void emit_build() {
    const BuildDecl* bd = nullptr;
    for (auto& b : prog.builds)
      if (b.adt == plan.adt->name) bd = &b;
    out << "  static constexpr bool kHasBuild = " << (bd ? "true" : "false") << ";  // build_node(): the layout's `build` block, compiled\n";
    if (!bd) return;
    const bool post = bd->order == "post";
    out << "  static constexpr bool kBuildPost = " << (post ? "true" : "false") << ";\n";
    const std::string self = "L_" + ident_of(plan.layout_name);
    const std::string this_t = ctype(plan.ref[0].type);
    in_build = true;
    for (auto& c : bd->ctors) {
      const Variant* v = find_variant(c.variant);
      if (!v) throw LayoutError("build block names unknown variant " + c.variant);
      auto hit = plan.variant_home.find(c.variant);
      const int home = hit == plan.variant_home.end() ? -1 : hit->second;
      const Buffer* hb = home >= 0 ? &plan.buffers[(size_t)home] : nullptr;
      // helper funcs the constructor reaches are emitted with the decode helpers (reach() in run())
      out << "  template <class B>\n  static uint64_t build_" << c.variant << "(B& b__, const typename B::Node& n__) {\n";
      out << "    using Self__ = " << self << ";\n";
      if (hb)
        for (size_t sg = 0; sg < hb->segments.size(); sg++)
          out << "    uint32_t rec" << sg << "__[" << (hb->segments[sg].stride_bytes + 3) / 4 + 1 << "] = {0};\n";
      for (auto& pa : c.params) {
        if (is_child_type(pa.type)) continue;                                   // children are built, not read
        if (pa.type->kind == Type::Array && !pa.type->len_field.empty()) continue;  // data: only `append` touches it
        out << "    const " << ctype(pa.type) << " " << pa.name << " = (" << ctype(pa.type) << ")n__." << pa.name << ";\n";
      }
      auto reserve = [&]() {
        if (!hb) { out << "    const " << this_t << " this__ = 0;\n"; return; }
        uint64_t bytes = hb->segments[0].stride_bytes;
        if (hb->is_arena) bytes = (bytes + hb->align - 1) / hb->align * hb->align;
        out << "    const " << this_t << " this__ = (" << this_t << ")b__.reserve(" << hb->id << ", " << bytes << "ull);\n";
      };
      size_t last_child = 0;
      bool any_child = false;
      for (size_t i = 0; i < c.body.size(); i++)
        if (stmt_builds_child(c.body[i], c)) { last_child = i; any_child = true; }
      if (!post || !any_child) reserve();
      // globals the statements outside the root block read
      std::set<std::string> ids;
      std::function<void(const std::vector<StmtP>&)> scan = [&](const std::vector<StmtP>& b) {
        for (auto& st : b) {
          if (st->kind == Stmt::BuildRoot) continue;
          collect_idents(st->value, ids);
          collect_idents(st->cond, ids);
          scan(st->then_body);
          scan(st->else_body);
        }
      };
      scan(c.body);
      std::set<std::string> param_names;
      for (auto& pa : c.params) param_names.insert(pa.name);
      auto read_globals = [&]() {
        for (size_t g = 0; g < plan.globals.size(); g++)
          if (ids.count(plan.globals[g].name) && !plan.globals[g].inferred && !param_names.count(plan.globals[g].name))
            out << "    const " << ctype(plan.globals[g].type) << " " << plan.globals[g].name << " = b__.template glob<" << ctype(plan.globals[g].type) << ">(" << g << ");\n";
      };
      bool has_root_block = false;
      for (auto& st : c.body)
        if (st->kind == Stmt::BuildRoot) has_root_block = true;
      if (!has_root_block) read_globals();
      std::function<void(const StmtP&, const std::string&, bool)> emit_build_stmt = [&](const StmtP& st, const std::string& pad, bool in_root) {
        const std::string& n = st->name;
        // the value: the expression, or the same-named constructor parameter
        bool child_param = false;
        TypeP ptype;
        for (auto& pa : c.params)
          if (pa.name == n) { ptype = pa.type; child_param = is_child_type(pa.type); }
        const Slot* slot = nullptr;
        if (hb)
          for (auto& sl : plan.slots)
            if (sl.name == n && sl.buffer == hb->id) slot = &sl;
        if (!st->value && child_param) {  // `build left;` / `build children;`
          const bool many = ptype->kind == Type::Array || ptype->kind == Type::Vec;
          if (many) {
            out << pad << "scion::vec<uint64_t, " << ptype->lanes << "> " << n << "__refs;\n";
            out << pad << "for (int k__ = 0; k__ < " << ptype->lanes << "; k__++) " << n << "__refs[k__] = (uint64_t)b__.template child<Self__>(n__." << n << "[k__]);\n";
            if (slot) deposit(slot->type, slot->offset, "rec" + std::to_string(slot->segment) + "__", n + "__refs", pad);
          } else {
            out << pad << "const uint64_t " << n << "__ref = (uint64_t)b__.template child<Self__>(n__." << n << ");\n";
            if (slot) deposit(slot->type, slot->offset, "rec" + std::to_string(slot->segment) + "__", n + "__ref", pad);
            else out << pad << "(void)" << n << "__ref;\n";
          }
          return;
        }
        const std::string val = st->value ? ex(st->value, false) : n;
        if (slot) {
          out << pad << "{ const " << ctype(slot->type) << " v__ = (" << ctype(slot->type) << ")(" << val << ");\n";
          deposit(slot->type, slot->offset, "rec" + std::to_string(slot->segment) + "__", "v__", pad + "  ");
          out << pad << "}\n";
          return;
        }
        for (size_t g = 0; g < plan.globals.size(); g++)
          if (plan.globals[g].name == n) {
            if (!in_root) throw LayoutError("build of global '" + n + "' outside a root block");
            out << pad << "const " << ctype(plan.globals[g].type) << " " << n << " = (" << ctype(plan.globals[g].type) << ")(" << val << ");\n";
            out << pad << "b__.set_global(" << g << ", " << n << ");\n";
            return;
          }
        for (size_t r = 1; r < plan.ref.size(); r++)
          if (plan.ref[r].name == n) {  // tree-carried component of the root reference (shared-slab: plo, phi)
            if (!in_root) throw LayoutError("build of reference component '" + n + "' outside a root block");
            out << pad << "const " << ctype(plan.ref[r].type) << " " << n << " = (" << ctype(plan.ref[r].type) << ")(" << val << ");\n";
            out << pad << "b__.set_root_component(" << r << ", " << n << ");\n";
            for (size_t g = 0; g < plan.globals.size(); g++)
              if (plan.globals[g].name == "__ref_" + n) out << pad << "b__.set_global(" << g << ", " << n << ");\n";
            return;
          }
        throw LayoutError("layout " + plan.layout_name + ": `build " + n + "` names neither a stored field of variant " + c.variant + "'s record, a global, a reference component nor a child");
      };
      bool returned = false;
      for (size_t i = 0; i < c.body.size(); i++) {
        const StmtP& st = c.body[i];
        switch (st->kind) {
          case Stmt::BuildRoot:
            out << "    if (b__.is_root(n__)) {  // root block: runs once, before anything else of the build (SPEC.md:282)\n";
            for (auto& rs : st->then_body) {
              if (rs->kind == Stmt::Build) emit_build_stmt(rs, "      ", true);
              else emit_stmts({rs}, 3);
            }
            out << "    }\n";
            read_globals();
            break;
          case Stmt::Build: emit_build_stmt(st, "    ", false); break;
          case Stmt::Return: {
            if (!st->value) throw LayoutError("a constructor must return the node's reference");
            out << "    const uint64_t ret__ = (uint64_t)(" << ex(st->value, false) << ");\n";
            if (hb)
              for (size_t sg = 0; sg < hb->segments.size(); sg++)
                out << "    b__.commit(" << hb->id << ", " << sg << ", (uint64_t)this__, rec" << sg << "__, " << hb->segments[sg].stride_bytes << "ull);\n";
            out << "    return ret__;\n";
            returned = true;
            break;
          }
          default: emit_stmts({st}, 2); break;
        }
        if (post && any_child && i == last_child) reserve();
      }
      if (!returned) throw LayoutError("constructor of " + c.variant + " does not return");
      out << "  }\n";
    }
    out << "  template <class B>\n  static uint64_t build_node(B& b__, const typename B::Node& n__) {\n";
    for (size_t i = 0; i < bd->ctors.size(); i++) {
      out << "    " << (i ? "else " : "") << "if (n__.variant == " << variant_index(bd->ctors[i].variant) << ") return build_" << bd->ctors[i].variant << "(b__, n__);\n";
    }
    out << "    return 0;\n  }\n";
    in_build = false;
  }

  // ------------------------------------------------------------------ decode emission
  struct GroupInfo {
    const MemberNode* node = nullptr;
    const Buffer* buf = nullptr;
  };
  std::map<std::string, GroupInfo> indirect_groups;
  const MemberNode* primary = nullptr;
  const Buffer* primary_buf = nullptr;

  std::set<std::string> cold_names;  // stored fields behind `---` and everything depending on them
  bool split_is_cold(const MemberNode& m) const {
    std::set<std::string> ids;
    collect_idents(m.value, ids);
    for (auto& i : ids)
      if (cold_names.count(i)) return true;
    for (auto& a : m.arms)
      for (auto& am : a.members)
        if ((am->kind == MemberNode::Stored || am->kind == MemberNode::Derive || am->kind == MemberNode::Let) && cold_names.count(am->name)) return true;
    return false;
  }
  void compute_cold(const std::vector<MemberP>& ms) {
    // stored fields in segments >= 1
    for (auto& s : plan.slots)
      if (primary_buf && s.buffer == primary_buf->id && s.segment > 0) cold_names.insert(s.name);
    bool changed = true;
    std::function<void(const std::vector<MemberP>&)> pass = [&](const std::vector<MemberP>& v) {
      for (auto& m : v) {
        if ((m->kind == MemberNode::Derive || m->kind == MemberNode::Let) && !cold_names.count(m->name)) {
          std::set<std::string> ids;
          collect_idents(m->value, ids);
          for (auto& i : ids)
            if (cold_names.count(i)) { cold_names.insert(m->name); changed = true; break; }
        }
        if (m->kind == MemberNode::Split) {
          bool cold = split_is_cold(*m);
          for (auto& a : m->arms) {
            if (cold)
              for (auto& am : a.members)
                if (!am->name.empty() && !cold_names.count(am->name)) { cold_names.insert(am->name); changed = true; }
            pass(a.members);
          }
        }
      }
    };
    while (changed) {
      changed = false;
      pass(ms);
    }
  }

  int gcd_align(const Buffer& b, int segment) const {
    uint64_t g = 256;  // cudaMalloc'd sub-allocations are 256-byte aligned
    if (b.is_arena) return (int)std::gcd<uint64_t>(g, b.align);
    for (int s = 0; s <= segment; s++) g = std::gcd<uint64_t>(g, b.segments[(size_t)s].stride_bytes);
    if (segment > 0) g = std::gcd<uint64_t>(g, b.align > 1 ? b.align : g);
    return (int)g;
  }

  // emits loads of every segment of `buf` that holds a wanted stored field
  // `stageable`: segment 0 of the primary index-referenced group may be served from a staged copy
  // of the array's first records (TMA bulk copy into shared memory, device/traverse.cuh)
  void emit_record_loads(const Buffer& buf, const std::string& index_expr, const std::string& tag, int ind, bool hot_only, bool stageable = false) {
    std::string pad((size_t)ind * 2, ' ');
    for (size_t s = 0; s < buf.segments.size(); s++) {
      if (hot_only && s > 0) break;
      uint64_t bytes = buf.segments[s].stride_bytes;
      std::string w = "w_" + tag + std::to_string(s);
      out << pad << "scion::Words<" << (bytes + 3) / 4 << "> " << w << ";\n";
      std::ostringstream addr;
      addr << "tree__.buf[" << buf.id << "] + ";
      if (buf.is_arena) addr << "(uint64_t)(" << index_expr << ")";
      else if (s == 0) addr << "(uint64_t)(" << index_expr << ") * " << bytes << "ull";  // segment 0 starts at the buffer base (plan.cpp:333-347)
      else addr << "tree__.seg_base[" << buf.id << "][" << s << "] + (uint64_t)(" << index_expr << ") * " << bytes << "ull";
      if (stageable && s == 0 && !buf.is_arena) {
        out << pad << "if constexpr (STAGED) {\n";
        out << pad << "  const uint64_t i__ = (uint64_t)(" << index_expr << ");\n";
        out << pad << "  const uint8_t* p__ = i__ < stage__.count ? stage__.base + i__ * " << bytes << "ull : " << addr.str() << ";\n";
        out << pad << "  scion::load_record_generic<" << bytes << ", " << gcd_align(buf, (int)s) << ">(p__, " << w << ");\n";
        out << pad << "} else {\n";
        out << pad << "  scion::load_record<" << bytes << ", " << gcd_align(buf, (int)s) << ">(" << addr.str() << ", " << w << ");\n";
        out << pad << "}\n";
      } else {
        out << pad << "scion::load_record<" << bytes << ", " << gcd_align(buf, (int)s) << ">(" << addr.str() << ", " << w << ");\n";
      }
    }
  }

  enum class Mode { All, Hot, Cold };

  bool is_adt_field(const std::string& n, const Variant* v) const {
    for (auto& f : plan.adt->fields)
      if (f.name == n) return true;
    if (v)
      for (auto& f : v->fields)
        if (f.name == n) return true;
    return false;
  }
  const Variant* find_variant(const std::string& n) const {
    for (auto& v : plan.adt->variants)
      if (v.name == n) return &v;
    return nullptr;
  }
  int variant_index(const std::string& n) const {
    for (size_t i = 0; i < plan.adt->variants.size(); i++)
      if (plan.adt->variants[i].name == n) return (int)i;
    return -1;
  }

  // Emits one member list. `bound` accumulates the names visible so far (for ADT assignment);
  // `assigned` the ADT fields already written at an outer level.
  void emit_members(const std::vector<MemberP>& ms, const Buffer* buf, const std::string& tag, int ind, Mode mode,
                    std::set<std::string> bound, std::set<std::string> assigned, const Variant* variant, bool arm_level) {
    std::string pad((size_t)ind * 2, ' ');
    auto wanted = [&](const std::string& name) {
      bool cold = cold_names.count(name) > 0;
      return mode == Mode::All || (mode == Mode::Hot && !cold) || mode == Mode::Cold;
    };
    auto assign_ok = [&](const std::string& name) {
      bool cold = cold_names.count(name) > 0;
      return mode == Mode::All || (mode == Mode::Hot && !cold) || (mode == Mode::Cold && cold);
    };
    // 1. stored fields of this level
    for (auto& m : ms)
      if (m->kind == MemberNode::Stored && wanted(m->name)) {
        const Slot* s = nullptr;
        for (auto& sl : plan.slots)
          if (sl.member == m.get()) s = &sl;
        if (!s) throw LayoutError("internal: unplanned field " + m->name);
        if (mode == Mode::Hot && s->segment > 0) continue;
        out << pad << "const " << ctype(m->type) << " " << m->name << " = " << extract(m->type, s->offset, "w_" + tag + std::to_string(s->segment)) << ";\n";
        bound.insert(m->name);
      }
    // 2. lets / derives in dependency order
    std::vector<const MemberNode*> pend;
    for (auto& m : ms)
      if ((m->kind == MemberNode::Let || m->kind == MemberNode::Derive) && wanted(m->name)) pend.push_back(m.get());
    std::set<std::string> pend_names;
    for (auto* m : pend) pend_names.insert(m->name);
    while (!pend.empty()) {
      bool progress = false;
      for (size_t i = 0; i < pend.size(); i++) {
        std::set<std::string> ids;
        collect_idents(pend[i]->value, ids);
        bool ready = true;
        for (auto& id : ids)
          if (pend_names.count(id) && id != pend[i]->name) ready = false;
        if (!ready) continue;
        const MemberNode* m = pend[i];
        std::string ty = m->kind == MemberNode::Let ? ctype(m->type) : std::string("auto");
        if (m->kind == MemberNode::Derive) {  // derives of ADT fields get the field's type
          for (auto& f : plan.adt->fields)
            if (f.name == m->name) ty = ctype(f.type);
          if (variant)
            for (auto& f : variant->fields)
              if (f.name == m->name) ty = ctype(f.type);
        }
        out << pad << "const " << ty << " " << m->name << " = " << ex(m->value, true) << ";\n";
        bound.insert(m->name);
        pend_names.erase(m->name);
        pend.erase(pend.begin() + (long)i);
        progress = true;
        break;
      }
      if (!progress) throw LayoutError("cyclic derives in layout " + plan.layout_name);
    }
    // 3. ADT fields resolvable at this level
    auto assign_fields = [&](const std::vector<Param>& fs, bool variant_fields) {
      for (auto& f : fs)
        if (bound.count(f.name) && !assigned.count(f.name)) {
          // a variant's own field is written inside its arm: when the arm is only reached in the cold pass, a HOT stored
          // field it exposes (pbrt-soaos-align16: `nprims` sits with `low`, the split behind `---`) is written there too
          if (assign_ok(f.name) || (variant_fields && mode == Mode::Cold)) out << pad << "node__." << f.name << " = " << f.name << ";\n";
          assigned.insert(f.name);
        }
    };
    assign_fields(plan.adt->fields, false);
    if (arm_level && variant) {
      assign_fields(variant->fields, true);
      for (auto& f : variant->fields)
        if (!assigned.count(f.name) && !(mode == Mode::Hot && cold_names.count(f.name)))
          throw LayoutError("layout " + plan.layout_name + ": field '" + f.name + "' of variant " + variant->name + " is not defined");
      for (auto& f : plan.adt->fields)
        if (!assigned.count(f.name) && !(mode == Mode::Hot && cold_names.count(f.name)))
          throw LayoutError("layout " + plan.layout_name + ": field '" + f.name + "' is not defined for variant " + variant->name);
    }
    // 4. splits
    for (auto& m : ms) {
      if (m->kind != MemberNode::Split) continue;
      bool cold = split_is_cold(*m);
      if ((mode == Mode::Hot && cold)) continue;
      if (mode == Mode::Cold && !cold) continue;
      out << pad << "const auto disc__ = " << ex(m->value, true) << ";\n";
      for (size_t a = 0; a < m->arms.size(); a++) {
        const Arm& arm = m->arms[a];
        bool last = a + 1 == m->arms.size();
        std::string test;
        switch (arm.pat) {
          case Arm::Literal: test = "disc__ == " + std::to_string(arm.value); break;
          case Arm::Gt: test = "disc__ > " + std::to_string(arm.value); break;
          case Arm::Lt: test = "disc__ < " + std::to_string(arm.value); break;
          case Arm::Ge: test = "disc__ >= " + std::to_string(arm.value); break;
          case Arm::Le: test = "disc__ <= " + std::to_string(arm.value); break;
          case Arm::Wildcard: test = ""; break;
        }
        if (a == 0) out << pad << "if (" << test << ") {\n";
        else if (last || test.empty()) out << pad << "} else {" << (test.empty() ? "" : "  // " + test) << "\n";
        else out << pad << "} else if (" << test << ") {\n";
        const Variant* v = find_variant(arm.variant);
        if (!v) throw LayoutError("split arm names unknown variant " + arm.variant);
        std::string pad2 = pad + "  ";
        out << pad2 << "node__.variant = " << variant_index(arm.variant) << ";  // " << arm.variant << "\n";
        if (arm.is_from) {
          auto it = indirect_groups.find(arm.from_group);
          if (it == indirect_groups.end()) throw LayoutError("unknown indirect group " + arm.from_group);
          std::string t2 = ident_of(arm.from_group) + "_";
          out << pad2 << "const uint64_t key__ = (uint64_t)(" << ex(arm.from_key, true) << ");\n";
          emit_record_loads(*it->second.buf, "key__", t2, ind + 1, false);
          emit_members(it->second.node->members, it->second.buf, t2, ind + 1, Mode::All, bound, assigned, v, true);
        } else {
          emit_members(arm.members, buf, tag, ind + 1, mode == Mode::Cold ? Mode::Cold : mode, bound, assigned, v, true);
        }
      }
      out << pad << "}\n";
    }
  }

  void find_groups(const std::vector<MemberP>& ms) {
    for (auto& m : ms) {
      if (m->kind != MemberNode::Group) continue;
      const Buffer* b = nullptr;
      std::string nm = m->group_name;
      for (auto& bb : plan.buffers)
        if (!bb.is_global_array && (bb.name == nm || (nm.empty() && bb.name == "group" + std::to_string(bb.id)))) b = &bb;
      if (m->indirect) indirect_groups[m->group_name] = {m.get(), b};
      else if (!m->index_binding.empty() && !primary) { primary = m.get(); primary_buf = b; }
      find_groups(m->members);
    }
  }

  std::string run() {
    const std::string id = ident_of(plan.layout_name);
    for (auto& r : plan.ref) ref_names.insert(r.name);
    for (auto& g : plan.globals) global_names.insert(g.name);
    for (auto& b : plan.buffers)
      if (b.is_global_array) array_names.insert(b.name);
    ref_is_struct = plan.ref.size() > 1;
    find_groups(plan.layout->members);
    if (!primary) throw LayoutError("layout has no direct group indexed by a reference component");
    reach_members(plan.layout->members);
    for (auto& b : prog.builds)
      if (b.adt == plan.adt->name)
        for (auto& c : b.ctors) {
          std::vector<std::string> calls;
          collect_calls(c.body, calls);
          for (auto& f : calls)
            if (f != "append") reach(f);
        }
    if (primary_buf && primary_buf->segments.size() > 1) compute_cold(primary->members);
    bool has_cold = !cold_names.empty();

    out << "// GENERATED by scionc emit-cuda from layouts/" << id << ".scion — do not edit.\n";
    out << "// layout '" << plan.layout_name << "' : ADT " << plan.adt->name << ", family "
        << (plan.family == Family::Bvh2 ? "bvh2" : plan.family == Family::Dop14 ? "dop14" : "bvh8") << ", node group '" << plan.node_group << "'\n";
    out << "#pragma once\n#include \"../device/scion_rt.cuh\"\n\nnamespace scion_gen {\n\nstruct L_" << id << " {\n";
    out << "  static constexpr const char* kName = \"" << plan.layout_name << "\";\n";
    out << "  static constexpr int kFamily = " << (int)plan.family << ";\n";
    out << "  static constexpr uint32_t kMaxLeaf = " << plan.max_leaf << "u;\n";
    out << "  static constexpr bool kHasCold = " << (has_cold ? "true" : "false") << ";\n";
    // the bounds the box test reads (chrt.scion:4 `node.low`, `node.high`) sit behind `---`: the traversal must read the
    // cold segment BEFORE the test (pbrt-soaos-align16: {low, nprims} | {high, topology})
    const bool bounds_cold = plan.family == Family::Bvh2 && (cold_names.count("low") || cold_names.count("high"));
    out << "  static constexpr bool kBoundsCold = " << (bounds_cold ? "true" : "false") << ";\n";
    // buffers, records, slots
    for (auto& b : plan.buffers) {
      out << "  // buffer " << b.id << ": " << b.name << (b.is_arena ? " (arena, byte-offset references)" : b.is_global_array ? " (global array)" : "")
          << ", count '" << b.count_name << "', align " << b.align << "\n";
      out << "  static constexpr int kBuf_" << ident_of(b.name) << " = " << b.id << ";\n";
      out << "  static constexpr uint32_t kStride_" << ident_of(b.name) << " = " << b.node_stride() << "u;\n";
    }
    // the device node record(s): typed, packed, one struct per segment (emit_records.cpp)
    {
      std::istringstream rec(emit_records(plan, "Record_", false));
      std::string line;
      while (std::getline(rec, line)) out << "  " << line << "\n";
    }
    for (auto& s : plan.slots)
      out << "  static constexpr uint32_t kOff_" << s.name << " = " << s.offset << "u, kWidth_" << s.name << " = " << s.width << "u, kSeg_" << s.name << " = " << s.segment << "u;  // "
          << s.type->str() << " in buffer " << s.buffer << "\n";
    for (size_t g = 0; g < plan.globals.size(); g++) out << "  static constexpr int kGlobal_" << plan.globals[g].name << " = " << g << ";  // " << plan.globals[g].type->str() << "\n";
    // record types
    for (auto& t : prog.types) {
      if (t.is_adt() || t.name == "Triangle") continue;
      out << "  struct rec_" << t.name << " {";
      for (auto& f : t.fields) out << " " << ctype(f.type) << " " << f.name << ";";
      out << " };\n";
    }
    // reference type
    if (ref_is_struct) {
      out << "  struct Ref {";
      for (auto& r : plan.ref) out << " " << ctype(r.type) << " " << r.name << ";";
      out << " };\n";
    } else {
      out << "  using Ref = " << ctype(plan.ref[0].type) << ";\n";
    }
    out << "  static constexpr uint32_t kRefBits = " << plan.type_bits(plan.ref[0].type) << "u;\n";
    for (size_t v = 0; v < plan.adt->variants.size(); v++) out << "  static constexpr int k" << plan.adt->variants[v].name << " = " << v << ";\n";
    // ADT view
    out << "  struct Node {\n    int variant;\n";
    std::set<std::string> seen;
    auto node_field = [&](const Param& f) {
      if (seen.count(f.name)) return;
      seen.insert(f.name);
      out << "    " << ctype(f.type) << " " << f.name << ";\n";
    };
    for (auto& f : plan.adt->fields) node_field(f);
    for (auto& v : plan.adt->variants)
      for (auto& f : v.fields) node_field(f);
    out << "  };\n";
    // root reference
    out << "  SCION_HOSTDEV static Ref root(const scion::TreeView& tree__) {\n";
    if (ref_is_struct) {
      out << "    Ref r;\n    r." << plan.ref[0].name << " = (" << ctype(plan.ref[0].type) << ")tree__.root0;\n";
      int k = 0;
      for (size_t i = 1; i < plan.ref.size(); i++) {
        const TypeP& t = plan.ref[i].type;
        if (t->kind == Type::Vec && t->elem->kind == Type::Float) {
          for (uint32_t l = 0; l < t->lanes; l++) out << "    r." << plan.ref[i].name << "[" << l << "] = tree__.root_carried[" << k++ << "];\n";
        } else if (t->kind == Type::Float) {
          out << "    r." << plan.ref[i].name << " = tree__.root_carried[" << k++ << "];\n";
        } else {
          throw LayoutError("unsupported tree-carried reference component type " + t->str());
        }
      }
      out << "    return r;\n";
    } else {
      out << "    return (Ref)tree__.root0;\n";
    }
    out << "  }\n";
    // ref_variant(): where the primary split discriminates on the reference alone (reference-encoded
    // variants, e.g. every 8-wide layout of the corpus) the traversal can tell a leaf reference from an
    // interior one without touching memory
    {
      const MemberNode* split = nullptr;
      for (auto& m : primary->members)
        if (m->kind == MemberNode::Split && !split) split = m.get();
      bool in_ref = split != nullptr;
      if (split) {
        std::set<std::string> ids;
        collect_idents(split->value, ids);
        for (auto& id : ids)
          if (!ref_names.count(id)) in_ref = false;
      }
      out << "  static constexpr bool kVariantInRef = " << (in_ref ? "true" : "false") << ";\n";
      out << "  SCION_HOSTDEV static int ref_variant(const Ref& ref__) {\n";
      if (in_ref) {
        out << "    const auto disc__ = " << ex(split->value, true) << ";\n";
        for (size_t a = 0; a < split->arms.size(); a++) {
          const Arm& arm = split->arms[a];
          std::string test;
          switch (arm.pat) {
            case Arm::Literal: test = "disc__ == " + std::to_string(arm.value); break;
            case Arm::Gt: test = "disc__ > " + std::to_string(arm.value); break;
            case Arm::Lt: test = "disc__ < " + std::to_string(arm.value); break;
            case Arm::Ge: test = "disc__ >= " + std::to_string(arm.value); break;
            case Arm::Le: test = "disc__ <= " + std::to_string(arm.value); break;
            case Arm::Wildcard: test = ""; break;
          }
          if (a + 1 == split->arms.size() || test.empty()) { out << "    return " << variant_index(arm.variant) << ";  // " << arm.variant << "\n"; break; }
          out << "    if (" << test << ") return " << variant_index(arm.variant) << ";  // " << arm.variant << "\n";
        }
      } else {
        out << "    (void)ref__;\n    return -1;  // the variant is stored in the node record\n";
      }
      out << "  }\n";
    }
    // helper funcs
    for (auto& fn : func_order) {
      const Func* f = find_func(fn);
      cur_ret = f->ret ? ctype(f->ret) : "void";
      out << "  SCION_HOSTDEV static " << cur_ret << " fn_" << f->name << "(";
      for (size_t i = 0; i < f->params.size(); i++) out << (i ? ", " : "") << ctype(f->params[i].type) << " " << f->params[i].name;
      out << ") {\n";
      emit_stmts(f->body, 2);
      out << "  }\n";
    }
    // decode
    const bool can_stage = primary_buf && !primary_buf->segments.empty() && !primary_buf->is_arena && primary_buf->segments[0].stride_bytes % 16 == 0;
    out << "  static constexpr bool kCanStage = " << (can_stage ? "true" : "false") << ";  // first records may be staged in shared memory\n";
    out << "  static constexpr uint32_t kStageStride = " << (can_stage ? primary_buf->segments[0].stride_bytes : 0) << "u;\n";
    out << "  static constexpr int kStageBuffer = " << (can_stage ? primary_buf->id : 0) << ";\n";
    // split form of decode() for single-segment records fetched by one vector load: fetch() issues the load, decode_fetched()
    // consumes the words later — lets a kernel keep a record in flight while it works on something else
    const bool can_fetch = can_stage && !has_cold;
    out << "  static constexpr bool kCanFetch = " << (can_fetch ? "true" : "false") << ";  // fetch() + decode_fetched() == decode()\n";
    if (can_fetch) {
      const Buffer& b = *primary_buf;
      const uint64_t bytes = b.segments[0].stride_bytes;
      std::string index_expr = ref_is_struct ? "ref__." + primary->index_binding : std::string("ref__");
      out << "  using Fetched = scion::Words<" << (bytes + 3) / 4 << ">;\n";
      const bool one_vector = (bytes == 16 && gcd_align(b, 0) % 16 == 0) || (bytes == 32 && gcd_align(b, 0) % 32 == 0);
      out << "  template <bool COLD = false>  // COLD: do not allocate the line in L1\n";
      out << "  SCION_HOSTDEV static void fetch(const scion::TreeView& tree__, const Ref& ref__, Fetched& w_0) {\n";
      out << "    const uint8_t* p__ = tree__.buf[" << b.id << "] + (uint64_t)(" << index_expr << ") * " << bytes << "ull;\n";
      if (one_vector) {
        out << "    if constexpr (COLD) scion::load_record_na<" << bytes << ", " << gcd_align(b, 0) << ">(p__, w_0);\n";
        out << "    else scion::load_record<" << bytes << ", " << gcd_align(b, 0) << ">(p__, w_0);\n";
      } else {
        out << "    scion::load_record<" << bytes << ", " << gcd_align(b, 0) << ">(p__, w_0);\n";
      }
      out << "  }\n";
    }
    auto emit_decode = [&](const char* name, Mode mode) {
      const bool main = std::string(name) == "decode";
      const bool fetched = std::string(name) == "decode_fetched";
      if (main) out << "  template <bool STAGED = false>\n";
      out << "  SCION_HOSTDEV static void " << name << "(const scion::TreeView& tree__, const Ref& ref__, " << (fetched ? "const Fetched& w_0, " : "") << "Node& node__"
          << (main ? ", const scion::Stage& stage__ = scion::Stage()" : "") << ") {\n";
      // globals referenced by layout expressions
      std::set<std::string> ids;
      std::function<void(const std::vector<MemberP>&)> scan = [&](const std::vector<MemberP>& ms) {
        for (auto& m : ms) {
          collect_idents(m->value, ids);
          scan(m->members);
          for (auto& a : m->arms) {
            collect_idents(a.from_key, ids);
            scan(a.members);
          }
        }
      };
      scan(plan.layout->members);
      for (size_t g = 0; g < plan.globals.size(); g++)
        if (ids.count(plan.globals[g].name) && !plan.globals[g].inferred)
          out << "    const " << ctype(plan.globals[g].type) << " " << plan.globals[g].name << " = scion::glob<" << ctype(plan.globals[g].type) << ">(tree__, " << g << ");\n";
      std::string index_expr = ref_is_struct ? "ref__." + primary->index_binding : std::string("ref__");
      if (primary_buf && !primary_buf->segments.empty() && !fetched) emit_record_loads(*primary_buf, index_expr, "", 2, mode == Mode::Hot, main && can_stage);
      emit_members(primary->members, primary_buf, "", 2, mode, {}, {}, nullptr, false);
      out << "  }\n";
    };
    if (has_cold) {
      emit_decode("decode", Mode::Hot);
      emit_decode("decode_cold", Mode::Cold);
    } else {
      emit_decode("decode", Mode::All);
      if (can_fetch) emit_decode("decode_fetched", Mode::All);
      out << "  SCION_HOSTDEV static void decode_cold(const scion::TreeView&, const Ref&, Node&) {}\n";
    }
    // Per-slot form of an 8-wide interior decode: decode_slot<K>() computes child slot K only, from ANY word source
    // (registers, or a lane's copy of the record staged in shared memory by 16-byte async copies — the extraction
    // templates of scion_rt.cuh are generic over the source).  It is the member list of the indirect group, emitted once
    // more; everything that does not feed slot K is dead code for the C++ compiler.  Emitted for records that start on a
    // 16-byte boundary (the `-align16` files and the 256-byte f32 record): that is what a 16-byte cp.async needs.
    {
      const MemberNode* from_split = nullptr;
      const Arm* from_arm = nullptr;
      if (plan.family == Family::Bvh8)
        for (auto& m : primary->members)
          if (m->kind == MemberNode::Split)
            for (auto& a : m->arms)
              if (a.is_from && !from_arm) { from_split = m.get(); from_arm = &a; }
      const GroupInfo* gi = nullptr;
      if (from_arm) {
        auto it = indirect_groups.find(from_arm->from_group);
        if (it != indirect_groups.end() && it->second.buf && it->second.buf->segments.size() == 1 && !it->second.buf->is_arena) gi = &it->second;
      }
      const bool can_slot = gi && gi->buf->segments[0].stride_bytes % 16 == 0;
      out << "  static constexpr bool kCanSlot = " << (can_slot ? "true" : "false") << ";  // 16-byte aligned interior record: may be staged by 16-byte async copies\n";
      // Per-child view of the record (scion::LaneRecord, lane-cooperative traversal: lane k of a group of 8 decodes child slot k
      // only): every stored field is either shared by all children (mlo, mex) or an 8-element array with one whole-byte element
      // per child (child_bounds, children, lo, hi).  The table gives [begin, end) bit offsets and the element width of each.
      struct LaneField { uint64_t off, end; uint64_t elem; };
      std::vector<LaneField> lane_fields;
      bool can_lane = gi != nullptr;
      if (gi) {
        for (auto& sl : plan.slots) {
          if (sl.buffer != gi->buf->id || sl.segment != 0) continue;
          uint64_t elem = 0;
          if (sl.type && (sl.type->kind == Type::Vec || sl.type->kind == Type::Array) && sl.type->lanes == 8 && sl.type->len_field.empty()) {
            elem = sl.width / 8;
            if (sl.width % 8 != 0 || elem % 8 != 0 || sl.offset % 8 != 0) can_lane = false;
          }
          lane_fields.push_back(LaneField{sl.offset, sl.offset + sl.width, elem});
        }
        if (lane_fields.empty()) can_lane = false;
      }
      out << "  static constexpr bool kCanLane = " << (can_lane ? "true" : "false") << ";  // per-child view of the interior record (scion::LaneRecord)\n";
      if (gi) {
        const Buffer& b = *gi->buf;
        const uint64_t bytes = b.segments[0].stride_bytes;
        const Variant* v = find_variant(from_arm->variant);
        std::string t2 = ident_of(from_arm->from_group) + "_";
        out << "  static constexpr uint32_t kSlotRecordBytes = " << bytes << "u;  // stride of the interior record\n";
        out << "  static constexpr uint32_t kSlotUsedBytes = " << (b.segments[0].stride_bits + 7) / 8 << "u;  // bytes the fields occupy (the rest is alignment padding)\n";
        if (can_lane) {
          out << "  static constexpr uint32_t kLaneAlign = " << gcd_align(b, 0) << "u;  // alignment every record address is known to have\n";
          out << "  static constexpr int kLaneFields = " << lane_fields.size() << ";\n";
          auto table = [&](const char* name, auto get, const char* what) {
            out << "  static constexpr uint32_t " << name << "[" << lane_fields.size() << "] = {";
            for (size_t i = 0; i < lane_fields.size(); i++) out << (i ? ", " : "") << get(lane_fields[i]) << "u";
            out << "};  // " << what << "\n";
          };
          table("kLaneFieldOff", [](const LaneField& f) { return f.off; }, "first bit of each stored field");
          table("kLaneFieldEnd", [](const LaneField& f) { return f.end; }, "one past its last bit");
          table("kLaneFieldElem", [](const LaneField& f) { return f.elem; }, "bits of one per-child element (0: the field is shared by all 8 children)");
        }
        out << "  SCION_HOSTDEV static const uint8_t* slot_record(const scion::TreeView& tree__, const Ref& ref__) {  // address of the interior record `ref__` designates\n";
        out << "    return tree__.buf[" << b.id << "] + (uint64_t)(" << ex(from_arm->from_key, true) << ") * " << bytes << "ull;\n  }\n";
        out << "  template <int K, class Src>\n";
        out << "  SCION_HOSTDEV static void decode_slot(const scion::TreeView& tree__, const Ref& ref__, const Src& w_" << t2 << "0, scion::vec<float, 3>& lo__, scion::vec<float, 3>& hi__, Ref& child__) {\n";
        out << "    (void)tree__; (void)ref__;\n";
        out << "    Node node__;\n";
        std::set<std::string> ids;
        std::function<void(const std::vector<MemberP>&)> scan = [&](const std::vector<MemberP>& ms) {
          for (auto& m : ms) {
            collect_idents(m->value, ids);
            scan(m->members);
          }
        };
        scan(gi->node->members);
        for (size_t g = 0; g < plan.globals.size(); g++)
          if (ids.count(plan.globals[g].name) && !plan.globals[g].inferred)
            out << "    const " << ctype(plan.globals[g].type) << " " << plan.globals[g].name << " = scion::glob<" << ctype(plan.globals[g].type) << ">(tree__, " << g << ");\n";
        emit_members(gi->node->members, gi->buf, t2, 2, Mode::All, {}, {}, v, true);
        out << "    lo__ = node__.lo[K];\n    hi__ = node__.hi[K];\n    child__ = node__.children[K];\n  }\n";
        (void)from_split;
      }
    }
    emit_build();
    // prefetch(): pull the record a reference designates into L2 ahead of its visit (issued by the
    // traversal when the reference is pushed on the stack)
    out << "  template <int LEVEL = 2>  // 2: into L2 (a reference that was pushed); 1: into L1 (a record about to be visited)\n";
    out << "  SCION_HOSTDEV static void prefetch(const scion::TreeView& tree__, const Ref& ref__) {\n";
    {
      std::string index_expr = ref_is_struct ? "ref__." + primary->index_binding : std::string("ref__");
      if (primary_buf && !primary_buf->segments.empty()) {
        const Buffer& b = *primary_buf;
        out << "    scion::prefetch_to<LEVEL>(tree__.buf[" << b.id << "] + ";
        if (b.is_arena) out << "(uint64_t)(" << index_expr << ")";
        else out << "(uint64_t)(" << index_expr << ") * " << b.segments[0].stride_bytes << "ull";
        out << ");\n";
      } else {
        // reference-encoded variants: prefetch only the arm(s) that live in an indirect group
        for (auto& m : primary->members) {
          if (m->kind != MemberNode::Split) continue;
          out << "    const auto disc__ = " << ex(m->value, true) << ";\n";
          for (auto& arm : m->arms) {
            if (!arm.is_from || arm.pat != Arm::Literal) continue;
            auto it = indirect_groups.find(arm.from_group);
            if (it == indirect_groups.end() || !it->second.buf || it->second.buf->segments.empty()) continue;
            const Buffer& b = *it->second.buf;
            uint64_t stride = b.segments[0].stride_bytes;
            out << "    if (disc__ == " << arm.value << ") {\n";
            out << "      const uint8_t* p__ = tree__.buf[" << b.id << "] + (uint64_t)(" << ex(arm.from_key, true) << ") * " << stride << "ull;\n";
            for (uint64_t o = 0; o < stride; o += 128) out << "      scion::prefetch_to<LEVEL>(p__ + " << o << ");\n";
            if (stride % 128 != 0 && stride > 64) out << "      scion::prefetch_to<LEVEL>(p__ + " << stride - 1 << ");  // the record may straddle a line\n";
            out << "    }\n";
          }
        }
      }
    }
    out << "  }\n";
    out << "};\n\n}  // namespace scion_gen\n";
    return out.str();
  }
};

}  // namespace

std::string emit_cuda(const Plan& plan) {
  Emitter e(plan);
  return e.run();
}

}  // namespace scion::lc
