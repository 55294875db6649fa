// TEST INFRASTRUCTURE — not part of the product.
//
// ref_interp: runs the REFERENCE's own compiled traversal on a PhysicalTree produced by this
// repository's encoders.  The reference ships its compiler front-end, planner and destructor
// specialiser (`specialize_destructors`, /root/reference/proj/src/specialize.cpp:143) but only a
// 15-byte placeholder for the executor (src/interp.cpp), so this file supplies the one missing
// piece — an interpreter for the reference's lowered IR (include/layoutc/ir.hpp) — and links it
// against the reference's real TUs compiled in place into oracle/_ref/ (oracle/Makefile `make ref`).
// What comes from the reference, unmodified: parsing of the corpus (.scion), type checking, the
// memory plan (every slot offset the loads use), the lowering of `closest_hit` for the layout
// (decode expressions, order of evaluation, comparison strictness, short-circuits, which loads
// happen) and the bit reader (`read_bits_raw`, src/bits.cpp:7-19).  What is ours: the meaning of
// each IR op below (IEEE binary32 arithmetic with one rounding per op, `dot`/`cross`/`sum`
// association ((x+y)+z), min/max = fminf/fmaxf — the conventions SURVEY §8c lists as unpinned).
//
// tools/gen_ref_ir_golden.py drives it here (the only place /root/reference exists) and commits the
// answers as fixtures under tests/golden/ref_ir/, which pin BOTH the oracle and the CUDA kernels.
//
// Two builds (oracle/Makefile): `ref_interp` links the UNMODIFIED reference and serves closest_hit; `ref_interp_fx`
// links the reference with the dangling-`Frame&` bug of src/lower_internal.hpp:1073/:890 patched at build time (one
// token, throw-away copy) and serves closest_point, whose lowering the unpatched reference corrupts.
//
// usage: ref_interp <corpus-layout | @family:/abs/layout.scion> <chrt|cpq> <tree+queries.bin> <out.bin>
//        ref_interp --print-ir <corpus-layout> <chrt|cpq|cd>          (the lowered IR as text, for build-vs-build diffs)
#include <array>
#include <cfenv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "layoutc/bits.hpp"
#include "layoutc/corpus.hpp"
#include "layoutc/ir.hpp"
#include "layoutc/plan.hpp"
#include "layoutc/sema.hpp"
#include "layoutc/specialize.hpp"

using namespace layoutc;

namespace {

struct Val {
  enum K { Int, Flt, Bool, Agg, Opt, Slice } k = Int;
  uint64_t i = 0;  // Int (raw bits, zero-extended to its width) / Bool / Opt: has
  float f = 0;
  std::vector<Val> e;  // Agg elements / Opt payload (0 or 1)
  int buf = -1;        // Slice
  uint64_t begin = 0, len = 0;
  static Val I(uint64_t v) { Val x; x.k = Int; x.i = v; return x; }
  static Val F(float v) { Val x; x.k = Flt; x.f = v; return x; }
  static Val B(bool v) { Val x; x.k = Bool; x.i = v; return x; }
};

struct Tree {
  struct Buf { std::vector<uint8_t> data; uint64_t count = 0; std::vector<uint64_t> seg_base; };
  std::vector<Buf> bufs;
  std::map<std::string, std::array<uint8_t, 16>> globals;
  uint64_t root0 = 0;
  float carried[6] = {0, 0, 0, 0, 0, 0};
};

uint64_t mask(uint32_t w) { return w >= 64 ? ~0ull : ((1ull << w) - 1ull); }
int64_t sext(uint64_t v, uint32_t w) { return w >= 64 ? (int64_t)v : (int64_t)(v << (64 - w)) >> (64 - w); }

struct Interp {
  const LoweredProgram& lp;
  const MemoryPlan& plan;  // specialize_destructors leaves LoweredProgram::plan empty; the MemoryPlan it was given is authoritative
  const Program& prog;
  TypeTable types;
  const Tree& tree;
  uint64_t node_loads = 0;
  Interp(const LoweredProgram& l, const MemoryPlan& mp, const Program& p, const Tree& t) : lp(l), plan(mp), prog(p), types(p), tree(t) {}

  uint64_t width_of(const SemType& t) const {
    std::string err;
    uint64_t w = types.packed_width(t, &err);
    if (!w) throw std::runtime_error("unstorable type " + type_to_string(t) + ": " + err);
    return w;
  }
  // packed value of type t at bit position `bit` of `buf` (record fields / lanes in declaration order, LSB first)
  Val load_typed(const uint8_t* buf, uint64_t bit, const SemType& t) const {
    switch (t.kind) {
      case TypeKind::Int: return Val::I(read_bits_raw(buf, bit, t.width));
      case TypeKind::Bool: return Val::B(read_bits_raw(buf, bit, 1) != 0);
      case TypeKind::Ptr: return Val::I(read_bits_raw(buf, bit, 64));
      case TypeKind::Float: {
        if (t.width != 32) throw std::runtime_error("only f32 storage is used by the corpus");
        uint32_t u = (uint32_t)read_bits_raw(buf, bit, 32);
        float f;
        memcpy(&f, &u, 4);
        return Val::F(f);
      }
      case TypeKind::Vec:
      case TypeKind::Array: {
        Val a; a.k = Val::Agg;
        uint64_t w = width_of(*t.elem);
        for (uint32_t l = 0; l < t.lanes; l++) a.e.push_back(load_typed(buf, bit + l * w, *t.elem));
        return a;
      }
      case TypeKind::Tuple: {
        Val a; a.k = Val::Agg;
        uint64_t off = 0;
        for (auto& m : t.members) { a.e.push_back(load_typed(buf, bit + off, *m)); off += width_of(*m); }
        return a;
      }
      case TypeKind::Named: {
        const AdtDecl* d = types.lookup(t.name);
        if (!d || !d->is_record()) throw std::runtime_error("load of non-record named type " + t.name);
        Val a; a.k = Val::Agg;
        uint64_t off = 0;
        for (auto& f : d->common_fields) { a.e.push_back(load_typed(buf, bit + off, *f.type)); off += width_of(*f.type); }
        return a;
      }
      default: throw std::runtime_error("load of type " + type_to_string(t));
    }
  }

  struct Frame { std::vector<Val> locals; bool returned = false; Val ret; };

  static bool truth(const Val& v) { return v.i != 0; }

  Val bin_scalar(BinOp op, const Val& a, const Val& b, const SemType& rt, const SemType& at) const {
    const bool cmp = op == BinOp::Eq || op == BinOp::Ne || op == BinOp::Lt || op == BinOp::Gt || op == BinOp::Le || op == BinOp::Ge;
    if (a.k == Val::Flt || b.k == Val::Flt) {
      const float x = a.k == Val::Flt ? a.f : (float)a.i, y = b.k == Val::Flt ? b.f : (float)b.i;
      switch (op) {
        case BinOp::Add: return Val::F(x + y);
        case BinOp::Sub: return Val::F(x - y);
        case BinOp::Mul: return Val::F(x * y);
        case BinOp::Div: return Val::F(x / y);
        case BinOp::Eq: return Val::B(x == y);
        case BinOp::Ne: return Val::B(x != y);
        case BinOp::Lt: return Val::B(x < y);
        case BinOp::Gt: return Val::B(x > y);
        case BinOp::Le: return Val::B(x <= y);
        case BinOp::Ge: return Val::B(x >= y);
        default: throw std::runtime_error("float binop");
      }
    }
    if (a.k == Val::Bool && b.k == Val::Bool) {
      switch (op) {
        case BinOp::And: case BinOp::BitAnd: return Val::B(a.i && b.i);
        case BinOp::Or: case BinOp::BitOr: return Val::B(a.i || b.i);
        case BinOp::Eq: return Val::B(a.i == b.i);
        case BinOp::Ne: case BinOp::BitXor: return Val::B(a.i != b.i);
        default: throw std::runtime_error("bool binop");
      }
    }
    // integers: the operand type decides signedness of comparisons / shifts / division; the result wraps to its width
    const SemType& ot = at;
    const uint32_t ow = ot.kind == TypeKind::Int ? ot.width : 64;
    const bool sg = ot.kind == TypeKind::Int && ot.is_signed;
    const uint64_t x = a.i, y = b.i;
    if (cmp) {
      if (sg) {
        const int64_t sx = sext(x, ow), sy = sext(y, ow);
        switch (op) {
          case BinOp::Eq: return Val::B(sx == sy); case BinOp::Ne: return Val::B(sx != sy);
          case BinOp::Lt: return Val::B(sx < sy); case BinOp::Gt: return Val::B(sx > sy);
          case BinOp::Le: return Val::B(sx <= sy); default: return Val::B(sx >= sy);
        }
      }
      switch (op) {
        case BinOp::Eq: return Val::B(x == y); case BinOp::Ne: return Val::B(x != y);
        case BinOp::Lt: return Val::B(x < y); case BinOp::Gt: return Val::B(x > y);
        case BinOp::Le: return Val::B(x <= y); default: return Val::B(x >= y);
      }
    }
    const uint32_t rw = rt.kind == TypeKind::Int ? rt.width : 64;
    uint64_t r = 0;
    switch (op) {
      case BinOp::Add: r = x + y; break;
      case BinOp::Sub: r = x - y; break;
      case BinOp::Mul: r = x * y; break;
      case BinOp::Div: r = sg ? (uint64_t)(sext(x, ow) / sext(y, ow)) : x / y; break;
      case BinOp::Mod: r = sg ? (uint64_t)(sext(x, ow) % sext(y, ow)) : x % y; break;
      case BinOp::Shl: r = x << y; break;
      case BinOp::Shr: r = sg ? (uint64_t)(sext(x, ow) >> y) : x >> y; break;
      case BinOp::BitAnd: r = x & y; break;
      case BinOp::BitOr: r = x | y; break;
      case BinOp::BitXor: r = x ^ y; break;
      default: throw std::runtime_error("int binop");
    }
    return Val::I(r & mask(rw));
  }
  static const SemType& lane_type(const SemType& t) { return (t.kind == TypeKind::Vec || t.kind == TypeKind::Array) && t.elem ? *t.elem : t; }
  Val bin(BinOp op, const Val& a, const Val& b, const SemType& rt, const SemType& at, const SemType& bt) const {
    if (a.k == Val::Agg || b.k == Val::Agg) {  // lane-wise, scalars broadcast
      const size_t n = a.k == Val::Agg ? a.e.size() : b.e.size();
      Val r; r.k = Val::Agg;
      for (size_t l = 0; l < n; l++)
        r.e.push_back(bin(op, a.k == Val::Agg ? a.e[l] : a, b.k == Val::Agg ? b.e[l] : b, lane_type(rt), a.k == Val::Agg ? lane_type(at) : at, b.k == Val::Agg ? lane_type(bt) : bt));
      return r;
    }
    // the operand type that carries signedness: prefer the non-literal (wider) integer operand
    const SemType& ot = (at.kind == TypeKind::Int) ? ((bt.kind == TypeKind::Int && bt.width > at.width) ? bt : at) : bt;
    return bin_scalar(op, a, b, rt, ot);
  }

  static float dot3(const Val& a, const Val& b) { return ((a.e[0].f * b.e[0].f) + (a.e[1].f * b.e[1].f)) + (a.e[2].f * b.e[2].f); }
  static float rounded(int mode, float x, float y, char op) {
    volatile float a = x, b = y;
    const int old = fegetround();
    fesetround(mode);
    volatile float r = op == '*' ? a * b : op == '+' ? a + b : op == '-' ? a - b : a / b;
    fesetround(old);
    return r;
  }
  Val map2(const Val& a, const Val& b, float (*fn)(float, float)) const {
    if (a.k == Val::Agg || b.k == Val::Agg) {
      const size_t n = a.k == Val::Agg ? a.e.size() : b.e.size();
      Val r; r.k = Val::Agg;
      for (size_t l = 0; l < n; l++) r.e.push_back(map2(a.k == Val::Agg ? a.e[l] : a, b.k == Val::Agg ? b.e[l] : b, fn));
      return r;
    }
    if (a.k == Val::Int && b.k == Val::Int) throw std::runtime_error("integer min/max are not used by the corpus traversals");
    return Val::F(fn(a.k == Val::Flt ? a.f : (float)a.i, b.k == Val::Flt ? b.f : (float)b.i));
  }
  Val intrin(Intrinsic in, std::vector<Val>& a) const {
    switch (in) {
      case Intrinsic::Dot: return Val::F(dot3(a[0], a[1]));
      case Intrinsic::Cross: {
        const Val &x = a[0], &y = a[1];
        Val r; r.k = Val::Agg;
        r.e = {Val::F(x.e[1].f * y.e[2].f - x.e[2].f * y.e[1].f), Val::F(x.e[2].f * y.e[0].f - x.e[0].f * y.e[2].f), Val::F(x.e[0].f * y.e[1].f - x.e[1].f * y.e[0].f)};
        return r;
      }
      case Intrinsic::Select: {
        if (a[0].k == Val::Agg) {
          Val r; r.k = Val::Agg;
          for (size_t l = 0; l < a[0].e.size(); l++) r.e.push_back(truth(a[0].e[l]) ? (a[1].k == Val::Agg ? a[1].e[l] : a[1]) : (a[2].k == Val::Agg ? a[2].e[l] : a[2]));
          return r;
        }
        return truth(a[0]) ? a[1] : a[2];
      }
      case Intrinsic::Min: {
        if (a.size() == 1 && a[0].k == Val::Agg) { Val r = a[0].e[0]; for (size_t l = 1; l < a[0].e.size(); l++) r = map2(r, a[0].e[l], fminf); return r; }
        return map2(a[0], a[1], fminf);
      }
      case Intrinsic::Max: {
        if (a.size() == 1 && a[0].k == Val::Agg) { Val r = a[0].e[0]; for (size_t l = 1; l < a[0].e.size(); l++) r = map2(r, a[0].e[l], fmaxf); return r; }
        return map2(a[0], a[1], fmaxf);
      }
      case Intrinsic::Floorf: return map2(a[0], a[0], [](float x, float) { return floorf(x); });
      case Intrinsic::Ceilf: return map2(a[0], a[0], [](float x, float) { return ceilf(x); });
      case Intrinsic::Abs: return map2(a[0], a[0], [](float x, float) { uint32_t u; memcpy(&u, &x, 4); u &= 0x7fffffffu; float r; memcpy(&r, &u, 4); return r; });
      case Intrinsic::Sum: { float s = a[0].e[0].f; for (size_t l = 1; l < a[0].e.size(); l++) s = s + a[0].e[l].f; return Val::F(s); }
      case Intrinsic::All: { bool all = true; for (auto& x : a[0].e) all = all && truth(x); return Val::B(all); }
      case Intrinsic::FmulRd: return map2(a[0], a[1], [](float x, float y) { return rounded(FE_DOWNWARD, x, y, '*'); });
      case Intrinsic::FaddRd: return map2(a[0], a[1], [](float x, float y) { return rounded(FE_DOWNWARD, x, y, '+'); });
      case Intrinsic::FsubRd: return map2(a[0], a[1], [](float x, float y) { return rounded(FE_DOWNWARD, x, y, '-'); });
      case Intrinsic::FsubRu: return map2(a[0], a[1], [](float x, float y) { return rounded(FE_UPWARD, x, y, '-'); });
      case Intrinsic::FdivRd: return map2(a[0], a[1], [](float x, float y) { return rounded(FE_DOWNWARD, x, y, '/'); });
      case Intrinsic::FrcpRd: return map2(a[0], a[0], [](float x, float) { return rounded(FE_DOWNWARD, 1.0f, x, '/'); });
      default: throw std::runtime_error("intrinsic not used by traversals");
    }
  }
  Val cast_val(const Val& v, const SemType& to, const SemType& from) const {
    if (v.k == Val::Agg) {
      Val r; r.k = Val::Agg;
      for (auto& x : v.e) r.e.push_back(cast_val(x, lane_type(to), lane_type(from)));
      return r;
    }
    if (to.kind == TypeKind::Float) {
      if (v.k == Val::Flt) return v;
      const bool sg = from.kind == TypeKind::Int && from.is_signed;
      return Val::F(sg ? (float)sext(v.i, from.width) : (float)v.i);
    }
    if (to.kind == TypeKind::Int || to.kind == TypeKind::Ptr) {
      const uint32_t w = to.kind == TypeKind::Int ? to.width : 64;
      if (v.k == Val::Flt) return Val::I((to.is_signed ? (uint64_t)(int64_t)v.f : (uint64_t)v.f) & mask(w));  // truncation
      uint64_t x = v.i;
      if (from.kind == TypeKind::Int && from.is_signed) x = (uint64_t)sext(x, from.width);
      return Val::I(x & mask(w));
    }
    if (to.kind == TypeKind::Bool) return Val::B(v.k == Val::Flt ? v.f != 0.0f : v.i != 0);
    throw std::runtime_error("cast to " + type_to_string(to));
  }
  Val cast_bits(const Val& v, const SemType& to) const {
    if (v.k == Val::Agg) {
      Val r; r.k = Val::Agg;
      for (auto& x : v.e) r.e.push_back(cast_bits(x, lane_type(to)));
      return r;
    }
    if (to.kind == TypeKind::Float) {
      if (v.k == Val::Flt) return v;
      uint32_t u = (uint32_t)v.i; float f; memcpy(&f, &u, 4); return Val::F(f);
    }
    if (v.k == Val::Flt) { uint32_t u; memcpy(&u, &v.f, 4); return Val::I(u); }
    const uint32_t w = to.kind == TypeKind::Int ? to.width : 64;
    return Val::I(v.i & mask(w));
  }

  Val load_elem(int buffer, uint64_t index) const {
    const BufferDesc& bd = plan.buffers[(size_t)buffer];
    const Tree::Buf& b = tree.bufs[(size_t)buffer];
    if (index >= b.count) throw std::runtime_error("out-of-bounds element access (query error, SPEC.md:382)");
    const uint64_t stride = bd.segments[0].stride_bytes * 8;
    return load_typed(b.data.data(), index * stride, *bd.elem_type);
  }

  Val eval(const IrFunc& f, Frame& fr, int id) {
    const IrExpr& e = f.exprs[(size_t)id];
    switch (e.op) {
      case IrOp::ConstI: return Val::I(e.u0);
      case IrOp::ConstF: return Val::F((float)e.f0);
      case IrOp::ConstB: return Val::B(e.u0 != 0);
      case IrOp::ReadVar: return fr.locals[(size_t)e.i0];
      case IrOp::LoadSlot: {
        const Val idx = eval(f, fr, e.args[0]);
        const BufferDesc& bd = plan.buffers[(size_t)e.i0];
        const Tree::Buf& b = tree.bufs[(size_t)e.i0];
        uint64_t bit;
        if (bd.is_arena) bit = idx.i * 8 + e.u0;
        else bit = b.seg_base[(size_t)e.i1] * 8 + idx.i * bd.segments[(size_t)e.i1].stride_bytes * 8 + e.u0;
        if ((bit + e.u1 + 7) / 8 > b.data.size()) throw std::runtime_error("out-of-bounds slot access (query error, SPEC.md:382)");
        node_loads++;
        return load_typed(b.data.data(), bit, *e.type);
      }
      case IrOp::LoadGlobal: {
        auto it = tree.globals.find(lp.str(e.u0));
        if (it == tree.globals.end()) throw std::runtime_error("global '" + lp.str(e.u0) + "' is not in the tree file");
        return load_typed(it->second.data(), 0, *e.type);
      }
      case IrOp::LoadElem: return load_elem(e.i0, eval(f, fr, e.args[0]).i);
      case IrOp::Bin: {
        const BinOp op = (BinOp)e.i0;
        const Val a = eval(f, fr, e.args[0]);
        if ((op == BinOp::And || op == BinOp::Or) && a.k == Val::Bool) {  // logical and/or never reach the IR un-lowered with side effects; plain evaluation
          const Val b = eval(f, fr, e.args[1]);
          return Val::B(op == BinOp::And ? (truth(a) && truth(b)) : (truth(a) || truth(b)));
        }
        const Val b = eval(f, fr, e.args[1]);
        return bin(op, a, b, *e.type, *f.exprs[(size_t)e.args[0]].type, *f.exprs[(size_t)e.args[1]].type);
      }
      case IrOp::Un: {
        const Val a = eval(f, fr, e.args[0]);
        switch ((UnOp)e.i0) {
          case UnOp::Not: return Val::B(!truth(a));
          case UnOp::Neg: return a.k == Val::Flt ? Val::F(-a.f) : Val::I((0 - a.i) & mask(e.type->kind == TypeKind::Int ? e.type->width : 64));
          default: return Val::I((~a.i) & mask(e.type->kind == TypeKind::Int ? e.type->width : 64));
        }
      }
      case IrOp::Intrin: {
        std::vector<Val> a;
        for (int x : e.args) a.push_back(eval(f, fr, x));
        return intrin((Intrinsic)e.i0, a);
      }
      case IrOp::CallF: {
        std::vector<int> args(e.args.begin(), e.args.end());
        return call(f, fr, e.i0, args);
      }
      case IrOp::MakeAgg: {
        Val r; r.k = Val::Agg;
        for (int x : e.args) r.e.push_back(eval(f, fr, x));
        return r;
      }
      case IrOp::GetElem: {
        Val a = eval(f, fr, e.args[0]);
        if (a.k != Val::Agg || e.u0 >= a.e.size()) throw std::runtime_error("get of a non-aggregate / out of range");
        return a.e[(size_t)e.u0];
      }
      case IrOp::IndexDyn: {
        Val a = eval(f, fr, e.args[0]);
        const Val i = eval(f, fr, e.args[1]);
        if (a.k == Val::Slice) return load_elem(a.buf, a.begin + i.i);
        if (i.i >= a.e.size()) throw std::runtime_error("dynamic index out of range");
        return a.e[(size_t)i.i];
      }
      case IrOp::BitExtract: {
        const Val a = eval(f, fr, e.args[0]);
        return Val::I((a.i >> e.u0) & mask((uint32_t)(e.u1 - e.u0 + 1)));
      }
      case IrOp::CastVal: return cast_val(eval(f, fr, e.args[0]), *e.type, *f.exprs[(size_t)e.args[0]].type);
      case IrOp::CastBits: return cast_bits(eval(f, fr, e.args[0]), *e.type);
      case IrOp::OptNone: { Val r; r.k = Val::Opt; r.i = 0; return r; }
      case IrOp::OptSome: { Val r; r.k = Val::Opt; r.i = 1; r.e.push_back(eval(f, fr, e.args[0])); return r; }
      case IrOp::OptHas: return Val::B(eval(f, fr, e.args[0]).i != 0);
      case IrOp::OptVal: {
        Val o = eval(f, fr, e.args[0]);
        if (!o.i) throw std::runtime_error("val() of none (runtime-checked, ir.hpp)");
        return o.e[0];
      }
      case IrOp::MakeSlice: {
        Val r; r.k = Val::Slice;
        r.buf = e.i0;
        r.begin = eval(f, fr, e.args[0]).i;
        r.len = eval(f, fr, e.args[1]).i;
        return r;
      }
      default: throw std::runtime_error("IR op outside the traversal subset");
    }
  }

  // a call binds arguments to the callee's parameter locals; `mut` parameters are copied back into the
  // caller's variable on return (no aliasing can occur in the corpus traversals)
  Val call(const IrFunc& caller, Frame& fr, int func, const std::vector<int>& args) {
    const IrFunc& g = lp.funcs[(size_t)func];
    Frame nf;
    nf.locals.resize(g.local_types.size());
    for (size_t k = 0; k < g.params.size(); k++) nf.locals[(size_t)g.params[k].local] = eval(caller, fr, args[k]);
    exec_block(g, nf, g.body);
    for (size_t k = 0; k < g.params.size(); k++) {
      if (!g.params[k].is_mut) continue;
      const IrExpr& a = caller.exprs[(size_t)args[k]];
      if (a.op != IrOp::ReadVar) throw std::runtime_error("mut argument is not a variable");
      fr.locals[(size_t)a.i0] = nf.locals[(size_t)g.params[k].local];
    }
    return nf.ret;
  }

  void exec_block(const IrFunc& f, Frame& fr, const std::vector<int>& block) {
    for (int id : block) {
      if (fr.returned) return;
      const IrStmt& s = f.stmts[(size_t)id];
      switch (s.kind) {
        case IrStmtKind::Assign: fr.locals[(size_t)s.var] = eval(f, fr, s.e0); break;
        case IrStmtKind::AssignLane: {
          const uint64_t lane = eval(f, fr, s.e0).i;
          Val v = eval(f, fr, s.e1);
          Val& dst = fr.locals[(size_t)s.var];
          if (dst.k != Val::Agg || lane >= dst.e.size()) throw std::runtime_error("assign_lane out of range");
          dst.e[(size_t)lane] = v;
          break;
        }
        case IrStmtKind::Eval: (void)eval(f, fr, s.e0); break;
        case IrStmtKind::If: {
          bool taken = false;
          for (auto& c : s.clauses) {
            if (truth(eval(f, fr, c.cond))) { exec_block(f, fr, c.block); taken = true; break; }
          }
          if (!taken) exec_block(f, fr, s.block);
          break;
        }
        case IrStmtKind::ForSlice: {
          const Val sl = eval(f, fr, s.e0);
          if (sl.k != Val::Slice) throw std::runtime_error("for_slice over a non-slice");
          for (uint64_t k = 0; k < sl.len && !fr.returned; k++) {
            fr.locals[(size_t)s.var] = load_elem(sl.buf, sl.begin + k);
            exec_block(f, fr, s.block);
          }
          break;
        }
        case IrStmtKind::ForVec: {
          const Val v = eval(f, fr, s.e0);
          for (size_t k = 0; k < v.e.size() && !fr.returned; k++) {
            fr.locals[(size_t)s.var] = v.e[k];
            exec_block(f, fr, s.block);
          }
          break;
        }
        case IrStmtKind::ForRange: {
          const uint64_t a = eval(f, fr, s.e0).i, b = eval(f, fr, s.e1).i;
          for (uint64_t k = a; k < b && !fr.returned; k++) {
            fr.locals[(size_t)s.var] = Val::I(k);
            exec_block(f, fr, s.block);
          }
          break;
        }
        case IrStmtKind::Return:
          if (s.e0 >= 0) fr.ret = eval(f, fr, s.e0);
          fr.returned = true;
          return;
        case IrStmtKind::Call: {
          std::vector<int> args(s.args.begin(), s.args.end());
          (void)call(f, fr, s.i0, args);
          break;
        }
        case IrStmtKind::Trap: throw std::runtime_error("trap: " + lp.str(s.u0));
        default: throw std::runtime_error("IR statement outside the traversal subset");
      }
    }
  }
};

template <class T> T rd(std::ifstream& in) { T v{}; in.read((char*)&v, sizeof(T)); return v; }
std::string rds(std::ifstream& in) { uint32_t n = rd<uint32_t>(in); std::string s(n, 0); in.read(s.data(), n); return s; }

}  // namespace

int main(int argc, char** argv) {
  const bool print_only = argc >= 4 && std::string(argv[1]) == "--print-ir";
  if (!print_only && argc < 5) { std::cerr << "usage: ref_interp <corpus-layout> <chrt|cpq> <in.bin> <out.bin> | --print-ir <corpus-layout> <alg>\n"; return 2; }
  try {
    const std::string name = print_only ? argv[2] : argv[1], alg = print_only ? argv[3] : argv[2];
    SourceSet ss;
    // <corpus-layout>, or an authored layout file of this repository: "@<bvh2|dop14|bvh8>:/abs/path/layout.scion" — the
    // reference's own library + algorithm sources (same pairing rule as corpus_files_for_pair) with that layout file
    std::vector<std::string> files;
    if (!name.empty() && name[0] == '@') {
      const size_t colon = name.find(':');
      if (colon == std::string::npos) throw std::runtime_error("expected @<family>:<path>");
      const std::string fam = name.substr(1, colon - 1), path = name.substr(colon + 1);
      files.push_back("lib/geometry.scion");
      if (fam == "dop14") files.push_back("lib/dop.scion");
      if (alg == "chrt") files.push_back(fam == "bvh8" ? "alg/chrt8.scion" : fam == "dop14" ? "alg/chrt_dop14.scion" : "alg/chrt.scion");
      else if (alg == "cpq") files.push_back(fam == "dop14" ? "alg/cpq_dop14.scion" : "alg/cpq.scion");
      else throw std::runtime_error("unknown algorithm");
      files.push_back(path);
    } else {
      files = corpus_files_for_pair(name, alg);
    }
    ParseResult r = parse_corpus(files, &ss);
    if (!r.ok()) throw std::runtime_error("parse failed");
    Program program = std::move(r.program);
    LayoutSpec* layout = nullptr;
    for (auto& l : program.layouts) if (program.find_build(l.name)) layout = &l;
    if (!layout && !program.layouts.empty()) layout = &program.layouts.back();  // authored files carry no build block (the destructors do not need one)
    if (!layout) throw std::runtime_error("no layout");
    const AdtDecl* adt = layout_adt(program, *layout);
    if (!typecheck_traversal(program).empty()) throw std::runtime_error("typecheck_traversal reported diagnostics");
    if (!check_layout(*adt, *layout, program).empty()) throw std::runtime_error("check_layout reported diagnostics");
    MemoryPlan plan = plan_layout(*adt, *layout, program);
    LoweredProgram lp;
    specialize_destructors(program, plan, lp);
    if (print_only) { std::cout << print_ir(lp); return 0; }
    const bool cpq = alg == "cpq";
    const IrFunc* entry = lp.entry(alg == "chrt" ? "closest_hit" : cpq ? "closest_point" : alg);
    if (!entry) throw std::runtime_error("no entry point");

    // ---- tree + rays (written by tools/gen_ref_ir_golden.py from this repository's encoders)
    std::ifstream in(argv[3], std::ios::binary);
    if (rd<uint32_t>(in) != 0x54494353u) throw std::runtime_error("bad input file");
    Tree tree;
    const uint32_t nbuf = rd<uint32_t>(in);
    if (nbuf != plan.buffers.size()) throw std::runtime_error("buffer count differs from the reference plan");
    for (uint32_t b = 0; b < nbuf; b++) {
      Tree::Buf buf;
      const std::string bname = rds(in);
      if (bname != plan.buffers[b].name) throw std::runtime_error("buffer " + std::to_string(b) + " is '" + bname + "' here, '" + plan.buffers[b].name + "' in the reference plan");
      buf.count = rd<uint64_t>(in);
      const uint32_t ns = rd<uint32_t>(in);
      for (uint32_t s = 0; s < ns; s++) buf.seg_base.push_back(rd<uint64_t>(in));
      const uint64_t bytes = rd<uint64_t>(in);
      buf.data.resize(bytes + 16);  // read_bits_raw may touch a trailing partial word
      in.read((char*)buf.data.data(), (std::streamsize)bytes);
      // the reference's own size formula must agree with the encoder's
      if (!plan.buffers[b].is_arena) {
        std::vector<uint64_t> bases;
        const uint64_t want = buffer_bytes(plan.buffers[b], buf.count, &bases);
        if (want != bytes || bases != buf.seg_base) throw std::runtime_error("buffer '" + bname + "': size / segment bases disagree with the reference's buffer_bytes()");
      }
      tree.bufs.push_back(std::move(buf));
    }
    const uint32_t ng = rd<uint32_t>(in);
    for (uint32_t g = 0; g < ng; g++) {
      const std::string gname = rds(in);
      std::array<uint8_t, 16> raw;
      in.read((char*)raw.data(), 16);
      tree.globals[gname] = raw;
    }
    tree.root0 = rd<uint64_t>(in);
    for (float& c : tree.carried) c = rd<float>(in);
    const uint64_t nrays = rd<uint64_t>(in);
    std::vector<float> rays(nrays * 8);
    in.read((char*)rays.data(), (std::streamsize)(nrays * 32));
    if (!in) throw std::runtime_error("truncated input file");

    // ---- root reference = the layout's reference components (+ the tree handle the lowering appends)
    const IrParamInfo& pb = entry->params[1];
    const SemType& rt = *entry->local_types[(size_t)pb.local];
    Val root; root.k = Val::Agg;
    {
      int carried = 0;
      for (size_t m = 0; m < rt.members.size(); m++) {
        const SemType& ct = *rt.members[m];
        if (m == 0) root.e.push_back(Val::I(tree.root0));
        else if (ct.kind == TypeKind::Vec) { Val v; v.k = Val::Agg; for (uint32_t l = 0; l < ct.lanes; l++) v.e.push_back(Val::F(tree.carried[carried++])); root.e.push_back(v); }
        else if (ct.kind == TypeKind::Float) root.e.push_back(Val::F(tree.carried[carried++]));
        else root.e.push_back(Val::I(0));  // tree handle
      }
    }
    std::ofstream out(argv[4], std::ios::binary);
    Interp it(lp, plan, program, tree);
    const float inf = std::numeric_limits<float>::infinity();
    for (uint64_t q = 0; q < nrays; q++) {
      const float* p = &rays[q * 8];
      Interp::Frame fr;
      fr.locals.resize(entry->local_types.size());
      Val ray; ray.k = Val::Agg;  // Ray(origin, direction, tmax), geometry.scion:4-9
      Val o; o.k = Val::Agg; o.e = {Val::F(p[0]), Val::F(p[1]), Val::F(p[2])};
      Val d; d.k = Val::Agg; d.e = {Val::F(p[4]), Val::F(p[5]), Val::F(p[6])};
      ray.e = {o, d, Val::F(p[3])};
      float rec[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      if (cpq) {  // closest_point(p: Point, bvh, best: mut (f32, Point)), cpq.scion:3; Point(v: f32x3), geometry.scion:9
        Val pt; pt.k = Val::Agg; pt.e = {o};
        Val zero; zero.k = Val::Agg; zero.e = {Val::F(0), Val::F(0), Val::F(0)};
        Val bp; bp.k = Val::Agg; bp.e = {zero};
        Val best; best.k = Val::Agg; best.e = {Val::F(inf), bp};
        fr.locals[(size_t)entry->params[0].local] = pt;
        fr.locals[(size_t)entry->params[1].local] = root;
        fr.locals[(size_t)entry->params[2].local] = best;
        it.exec_block(*entry, fr, entry->body);
        const Val& b = fr.locals[(size_t)entry->params[2].local];
        rec[0] = b.e[0].f;
        for (int a = 0; a < 3; a++) rec[1 + a] = b.e[1].e[0].e[(size_t)a].f;
      } else {
        Val tri; tri.k = Val::Agg;  // best = (inf, <zero triangle>)
        for (int v = 0; v < 3; v++) { Val x; x.k = Val::Agg; x.e = {Val::F(0), Val::F(0), Val::F(0)}; tri.e.push_back(x); }
        Val best; best.k = Val::Agg; best.e = {Val::F(inf), tri};
        fr.locals[(size_t)entry->params[0].local] = ray;
        fr.locals[(size_t)entry->params[1].local] = root;
        fr.locals[(size_t)entry->params[2].local] = best;
        it.exec_block(*entry, fr, entry->body);
        const Val& b = fr.locals[(size_t)entry->params[2].local];
        rec[0] = b.e[0].f;
        for (int v = 0; v < 3; v++) for (int a = 0; a < 3; a++) rec[1 + 3 * v + a] = b.e[1].e[(size_t)v].e[(size_t)a].f;
      }
      out.write((const char*)rec, sizeof(rec));
    }
    std::cerr << "ref_interp: " << name << " x " << alg << ": " << nrays << " queries, " << it.node_loads << " slot loads\n";
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "ref_interp: " << e.what() << "\n";
    return 1;
  }
}
