// scionc — the layout compiler of the B200 backend.
//
// Reads the *layout language* of Scion (the `type`, `func` and `layout` declarations of a
// .scion file, and its `build` blocks: emit_cuda turns them into the generated constructors,
// host/encode.cpp holds the hand-written per-family encoders they are checked against), plans the physical memory (bit-exact with the reference planner,
// /root/reference/proj/src/plan.cpp:75-140, :174-241, :307-347) and emits, per layout, a
// CUDA header with the device node record, slot constants and the decode routine
// (emit_cuda — the sibling of the reference's emit_c slot).
//
// Written from scratch for this backend: one recursive-descent parser over a flat token
// vector, a value-typed AST, no sema pass (C++ overload resolution in the emitted code
// does the typing; the DSL is C-like enough for a 1:1 expression translation).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace scion::lc {

struct LayoutError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --------------------------------------------------------------------------------- types
struct Type;
using TypeP = std::shared_ptr<Type>;
struct Type {
  enum Kind { Int, Float, Bool, Ptr, Vec, Array, Named, Tuple } kind = Int;
  uint32_t width = 0;      // Int / Float
  bool is_signed = false;  // Int
  TypeP elem;              // Vec / Array
  uint32_t lanes = 0;      // Vec lanes, static Array count
  std::string len_field;   // dynamic Array: name of the global holding the count
  std::string name;        // Named
  std::vector<TypeP> members;  // Tuple
  std::string str() const;
};

// --------------------------------------------------------------------------------- expressions
struct Expr;
using ExprP = std::shared_ptr<Expr>;
struct Expr {
  enum Kind { IntLit, FloatLit, Ident, Binary, Unary, Call, Member, Index, Range, Cast, Construct, Brace, Tuple, BuildChild } kind = IntLit;  // BuildChild: `build left` in expression position (text = the child parameter)
  uint64_t ival = 0;
  bool has_u = false;       // integer literal carried a 'u' suffix
  std::string text;         // FloatLit spelling, Ident / Call / Member name, operator
  std::vector<ExprP> args;  // operands
  TypeP type;               // Cast target / Construct type
  bool bitcast = false;     // Cast: `to` (true) vs `as` (false)
  int line = 0;
};

struct Stmt;
using StmtP = std::shared_ptr<Stmt>;
struct Stmt {
  // Build / BuildRoot only occur in the constructors of a `build` block: `build X;`, `build X = e;` (name = X, value = e or
  // null) and `build root { ... }` (then_body; runs once, for the root node, before anything else: SPEC.md:282)
  enum Kind { Let, Assign, If, Return, ExprS, Build, BuildRoot } kind = Let;
  std::string name;  // Let, Build
  TypeP type;        // Let
  bool is_mut = false;
  ExprP lhs, value, cond;
  std::vector<StmtP> then_body, else_body;
};

struct Param {
  std::string name;
  TypeP type;
  ExprP default_value;
};

struct Func {
  std::string name;
  std::vector<Param> params;
  TypeP ret;
  std::vector<StmtP> body;
};

struct Variant {
  std::string name;
  std::vector<Param> fields;
};
struct TypeDecl {
  std::string name;
  std::vector<Param> fields;      // record fields, or the ADT's shared base fields
  std::vector<Variant> variants;  // empty => record
  bool is_adt() const { return !variants.empty(); }
};

// --------------------------------------------------------------------------------- layout members
struct MemberNode;
using MemberP = std::shared_ptr<MemberNode>;
struct Arm {
  enum Pat { Literal, Gt, Lt, Ge, Le, Wildcard } pat = Wildcard;
  int64_t value = 0;
  std::string variant;
  bool is_from = false;
  std::string from_group;
  ExprP from_key;
  std::vector<MemberP> members;
};
struct MemberNode {
  enum Kind { Stored, Derive, Let, Padding, Separator, Group, Split } kind = Stored;
  std::string name;
  TypeP type;
  ExprP value;  // Derive/Let expression, Split discriminant
  uint64_t padding_bits = 0;
  // group
  bool indirect = false;
  std::string group_name, index_binding;
  ExprP size_expr;
  uint64_t align = 0, tile = 0;
  std::vector<MemberP> members;
  std::vector<Arm> arms;
};

// `build ADT[order=pre|post] { build Variant(params) { statements }; ... }` — the constructors of a layout
// (SPEC.md:276-284 specialize_constructors)
struct BuildCtor {
  std::string variant;
  std::vector<Param> params;  // the logical fields of the variant, by name
  std::vector<StmtP> body;
};
struct BuildDecl {
  std::string adt;
  std::string order = "pre";
  std::vector<BuildCtor> ctors;
};

struct Layout {
  std::string name;  // the ADT it realises
  std::vector<Param> ref;
  std::vector<MemberP> members;
};

struct Program {
  std::vector<TypeDecl> types;
  std::vector<Func> funcs;
  std::vector<Layout> layouts;
  std::vector<std::string> build_orders;  // "pre"/"post" of each build block
  std::vector<BuildDecl> builds;
  const TypeDecl* find_type(const std::string& n) const {
    for (auto& t : types)
      if (t.name == n) return &t;
    return nullptr;
  }
};

// Parses one or more sources (concatenated compile set). A built-in prelude declares the
// primitive record `Triangle(p0, p1, p2: f32x3)` unless the sources declare it themselves.
Program parse_program(const std::vector<std::string>& sources);

// --------------------------------------------------------------------------------- memory plan
struct Slot {
  std::string name;
  int buffer = -1, segment = 0;
  uint64_t offset = 0;  // bit offset inside one element of the segment
  uint32_t width = 0;
  TypeP type;
  const MemberNode* member = nullptr;
};
struct Segment {
  uint64_t stride_bits = 0, stride_bytes = 0;
};
struct Buffer {
  int id = -1;
  std::string name;
  bool is_arena = false, is_global_array = false;
  uint32_t align = 1;
  std::vector<Segment> segments;
  std::string count_name;
  TypeP elem_type;
  uint64_t node_stride() const {
    uint64_t s = 0;
    for (auto& g : segments) s += g.stride_bytes;
    return s;
  }
  // byte size + segment bases for `count` elements (plan.cpp:333-347 rule)
  uint64_t bytes(uint64_t count, std::vector<uint64_t>* bases = nullptr) const;
};
struct Global {
  std::string name;
  TypeP type;
  bool inferred = false;  // element counts filled by the builder
};

enum class Family { Bvh2 = 0, Dop14 = 1, Bvh8 = 2 };

struct Plan {
  std::string layout_name;  // registry name, e.g. "pbrt-q16"
  const Program* program = nullptr;
  const Layout* layout = nullptr;
  const TypeDecl* adt = nullptr;
  Family family = Family::Bvh2;
  std::vector<Param> ref;
  std::vector<Buffer> buffers;
  std::vector<Global> globals;
  std::vector<Slot> slots;
  std::map<std::string, int> variant_home;
  std::string node_group;   // buffer whose stride is "the node size"
  std::string build_order;  // "pre" | "post"
  uint32_t max_leaf = 0;    // capacity of the Leaf nprims field

  const Buffer* buffer_named(const std::string& n) const {
    for (auto& b : buffers)
      if (b.name == n) return &b;
    return nullptr;
  }
  const Slot* slot_named(const std::string& n) const {
    for (auto& s : slots)
      if (s.name == n) return &s;
    return nullptr;
  }
  const Slot& slot(const std::string& n) const {
    const Slot* s = slot_named(n);
    if (!s) throw LayoutError("layout " + layout_name + ": no stored field '" + n + "'");
    return *s;
  }
  uint64_t type_bits(const TypeP& t) const;
  std::string to_json() const;
};

// Well-formedness (check.cpp): throws LayoutError tagged with the reference's diagnostic class
// ([DuplicateName], [MissingField], [NonExhaustiveSplit], [UnsupportedPattern]).  plan_layout runs it first.
void check_layout(const Program& program, const Layout& layout, const TypeDecl& adt);
Plan plan_layout(const Program& program, const std::string& registry_name);

// emit_cuda: deterministic CUDA header text for the planned layout.
std::string emit_cuda(const Plan& plan);
// typed packed record declarations (one struct per node-buffer segment) + static assertions; shared by emit_cuda and emit-c
std::string emit_records(const Plan& plan, const std::string& prefix, bool c11);
// `scionc emit-c`: C11 header with the packed records, their assertions and the slot table (record half)
std::string emit_c_records(const Plan& plan);
// op-count report of the layout's decode, per variant (`scionc stats`; SPEC.md:360 --dump-stats)
std::string decode_stats_json(const Plan& plan);
// C-identifier form of a registry name ("pbrt-q16" -> "pbrt_q16")
std::string ident_of(const std::string& registry_name);

}  // namespace scion::lc
