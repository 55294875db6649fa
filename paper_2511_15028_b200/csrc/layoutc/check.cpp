// Well-formedness of a layout specification — the slice of the reference's `check_layout`
// (/root/reference/proj/src/sema_layout.cpp; diagnostic codes of include/layoutc/diag.hpp:18-35) that
// the B200 backend needs before it plans and emits a decoder: a specification that passes here can
// be planned and its emitted CUDA compiles; one that does not is rejected with the reference's
// diagnostic class in brackets ([DuplicateName], [MissingField], [NonExhaustiveSplit],
// [UnsupportedPattern]; [CyclicDerive] is reported by the emitter's scheduling of derives).
// SPEC acceptance criterion 4 (mutation suite: deleted arms / fields, duplicated fields, 0 false
// accepts) is exercised by tests/test_layoutc.py::test_mutation_suite over the 16 shipped layouts.
#include <functional>
#include <set>

#include "layoutc.hpp"

namespace scion::lc {
namespace {

struct Checker {
  const Program& prog;
  const Layout& layout;
  const TypeDecl& adt;
  std::set<std::string> top;      // names visible everywhere: reference components, globals, global arrays
  std::set<std::string> funcs, types;

  static void idents(const ExprP& e, std::set<std::string>& ids) {
    if (!e) return;
    if (e->kind == Expr::Ident) ids.insert(e->text);
    for (auto& a : e->args) idents(a, ids);
  }
  static void type_names(const TypeP& t, std::set<std::string>& ids, std::set<std::string>& lens) {
    if (!t) return;
    if (t->kind == Type::Named) ids.insert(t->name);
    if (!t->len_field.empty()) lens.insert(t->len_field);
    type_names(t->elem, ids, lens);
    for (auto& m : t->members) type_names(m, ids, lens);
  }
  [[noreturn]] void fail(const char* code, const std::string& what) const {
    throw LayoutError("layout " + layout.name + ": " + what + " [" + code + "]");
  }
  bool builtin(const std::string& n) const {
    static const std::set<std::string> k = {"inf", "true", "false", "this", "parent", "none", "SENTINEL"};
    return k.count(n) != 0;
  }

  // names a member list declares at its own level (stored fields, derives, lets, group index bindings excluded)
  void declare(const std::vector<MemberP>& ms, std::set<std::string>& names) const {
    for (auto& m : ms) {
      if (m->kind == MemberNode::Stored || m->kind == MemberNode::Derive || m->kind == MemberNode::Let) {
        if (!names.insert(m->name).second) fail("DuplicateName", "'" + m->name + "' is defined twice in the same scope");
      }
    }
  }
  void use(const ExprP& e, const std::set<std::string>& scope, const std::string& where) const {
    std::set<std::string> ids;
    idents(e, ids);
    for (auto& id : ids)
      if (!scope.count(id) && !top.count(id) && !funcs.count(id) && !types.count(id) && !builtin(id))
        fail("MissingField", "'" + id + "' used by " + where + " is not a field, global, reference component or function");
  }
  void use_type(const TypeP& t, const std::set<std::string>& scope, const std::string& where) const {
    std::set<std::string> ids, lens;
    type_names(t, ids, lens);
    for (auto& id : ids)
      if (!types.count(id)) fail("MissingField", "unknown type '" + id + "' in " + where);
    for (auto& l : lens)
      if (!scope.count(l) && !top.count(l)) fail("MissingField", "array length '" + l + "' of " + where + " is not a stored field or global");
  }

  // variants an arm list produces; every arm's members are checked in the scope of the enclosing levels
  void members(const std::vector<MemberP>& ms, std::set<std::string> scope, std::set<std::string>& produced, bool in_group) const {
    declare(ms, scope);
    for (auto& m : ms) {
      switch (m->kind) {
        case MemberNode::Stored:
          use_type(m->type, scope, "field '" + m->name + "'");
          break;
        case MemberNode::Derive:
        case MemberNode::Let:
          use(m->value, scope, "'" + m->name + "'");
          if (m->type) use_type(m->type, scope, "'" + m->name + "'");
          break;
        case MemberNode::Group: {
          std::set<std::string> inner = scope;
          if (!m->index_binding.empty()) inner.insert(m->index_binding);
          use(m->size_expr, scope, "the size of group '" + m->group_name + "'");
          members(m->members, inner, produced, true);
          break;
        }
        case MemberNode::Split: {
          use(m->value, scope, "a split discriminant");
          if (m->arms.empty()) fail("NonExhaustiveSplit", "split without arms");
          std::set<std::string> seen_pat;
          for (auto& a : m->arms) {
            const std::string pat = std::to_string((int)a.pat) + ":" + std::to_string(a.value);
            if (!seen_pat.insert(pat).second) fail("UnsupportedPattern", "two arms of a split have the same pattern");
            bool known = false;
            for (auto& v : adt.variants) known |= v.name == a.variant;
            if (!known) fail("MissingField", "split arm names '" + a.variant + "', which is not a variant of " + adt.name);
            if (!produced.insert(a.variant).second && !a.is_from) {
              // the same variant from two arms is legal (e.g. > 0 and a wildcard); nothing to do
            }
            if (a.is_from) use(a.from_key, scope, "the key of a `from` arm");
            std::set<std::string> sub;
            members(a.members, scope, sub, in_group);
          }
          break;
        }
        default: break;
      }
    }
  }

  void run() {
    for (auto& f : prog.funcs) funcs.insert(f.name);
    for (auto& t : prog.types) types.insert(t.name);
    for (auto& r : layout.ref) {
      if (!top.insert(r.name).second) fail("DuplicateName", "reference component '" + r.name + "' is declared twice");
    }
    // top-level scalars / arrays are visible everywhere (they become globals and global arrays)
    std::set<std::string> level;
    for (auto& m : layout.members) {
      if (m->kind == MemberNode::Stored || m->kind == MemberNode::Derive || m->kind == MemberNode::Let) {
        if (!level.insert(m->name).second || top.count(m->name)) fail("DuplicateName", "'" + m->name + "' is defined twice at the top level of the layout");
      }
    }
    for (auto& n : level) top.insert(n);
    // indirect groups are visible by name to `from G[key]` arms
    std::function<void(const std::vector<MemberP>&)> groups = [&](const std::vector<MemberP>& ms) {
      for (auto& m : ms) {
        if (m->kind == MemberNode::Group && !m->group_name.empty()) {
          if (!top.insert("@group:" + m->group_name).second) fail("DuplicateName", "group '" + m->group_name + "' is declared twice");
        }
        groups(m->members);
        for (auto& a : m->arms) groups(a.members);
      }
    };
    groups(layout.members);
    std::set<std::string> produced;
    // the top level was declared above: check its members without re-declaring them
    std::set<std::string> scope;
    for (auto& m : layout.members) {
      std::vector<MemberP> one{m};
      if (m->kind == MemberNode::Stored) use_type(m->type, scope, "field '" + m->name + "'");
      else if (m->kind == MemberNode::Derive || m->kind == MemberNode::Let) use(m->value, scope, "'" + m->name + "'");
      else members(one, scope, produced, false);
    }
    for (auto& v : adt.variants)
      if (!produced.count(v.name)) fail("NonExhaustiveSplit", "no split arm produces variant '" + v.name + "'");
  }
};

}  // namespace

void check_layout(const Program& program, const Layout& layout, const TypeDecl& adt) {
  Checker c{program, layout, adt, {}, {}, {}};
  c.run();
}

}  // namespace scion::lc
