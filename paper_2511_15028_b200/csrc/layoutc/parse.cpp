// Lexer + recursive-descent parser for the layout-language subset of Scion.
// Grammar source of truth: the reference's parser (/root/reference/proj/src/parser.cpp:
// types :108-147, expressions :467-517, funcs :766-788, layout members :799-955) and lexer
// (src/lexer.cpp:60-140).  Re-implemented from the grammar, not translated.
#include <cctype>
#include <cstdlib>

#include "layoutc.hpp"

namespace scion::lc {

std::string Type::str() const {
  switch (kind) {
    case Int: return (is_signed ? "i" : "u") + std::to_string(width);
    case Float: return "f" + std::to_string(width);
    case Bool: return "bool";
    case Ptr: return "ptr";
    case Vec: return elem->str() + "x" + std::to_string(lanes);
    case Array: return elem->str() + "[" + (len_field.empty() ? std::to_string(lanes) : len_field) + "]";
    case Named: return name;
    case Tuple: {
      std::string s = "(";
      for (size_t i = 0; i < members.size(); i++) s += (i ? ", " : "") + members[i]->str();
      return s + ")";
    }
  }
  return "?";
}

namespace {

enum class T { End, Ident, Int, Float, Punct, Sep };
struct Tok {
  T kind = T::End;
  std::string text;  // ident / punct spelling / float spelling
  uint64_t ival = 0;
  std::string suffix;
  int line = 1;
};

std::vector<Tok> lex(const std::string& s) {
  std::vector<Tok> out;
  size_t i = 0;
  int line = 1;
  auto peek = [&](size_t k = 0) { return i + k < s.size() ? s[i + k] : '\0'; };
  while (i < s.size()) {
    char c = s[i];
    if (c == '\n') { line++; i++; continue; }
    if (isspace((unsigned char)c)) { i++; continue; }
    if (c == '/' && peek(1) == '/') { while (i < s.size() && s[i] != '\n') i++; continue; }
    if (c == '/' && peek(1) == '*') {
      i += 2;
      while (i < s.size() && !(s[i] == '*' && peek(1) == '/')) { if (s[i] == '\n') line++; i++; }
      i += 2;
      continue;
    }
    Tok t;
    t.line = line;
    if (isalpha((unsigned char)c) || c == '_') {
      size_t b = i;
      while (i < s.size() && (isalnum((unsigned char)s[i]) || s[i] == '_')) i++;
      t.kind = T::Ident;
      t.text = s.substr(b, i - b);
      out.push_back(t);
      continue;
    }
    if (isdigit((unsigned char)c)) {
      // binary spellings 0b'101, 0'b101, 0b101 (lexer.cpp:93-119)
      if (c == '0' && ((peek(1) == 'b' && (peek(2) == '\'' || peek(2) == '0' || peek(2) == '1')) || (peek(1) == '\'' && peek(2) == 'b'))) {
        i++;
        if (s[i] == '\'') i++;
        i++;  // b
        if (peek() == '\'') i++;
        uint64_t v = 0;
        while (peek() == '0' || peek() == '1') v = (v << 1) | (uint64_t)(s[i++] - '0');
        t.kind = T::Int;
        t.ival = v;
        while (i < s.size() && (isalnum((unsigned char)s[i]) || s[i] == '_')) t.suffix += s[i++];
        out.push_back(t);
        continue;
      }
      size_t b = i;
      while (isdigit((unsigned char)peek())) i++;
      bool is_float = false;
      if (peek() == '.' && isdigit((unsigned char)peek(1))) {
        is_float = true;
        i++;
        while (isdigit((unsigned char)peek())) i++;
      }
      if ((peek() == 'e' || peek() == 'E') && (isdigit((unsigned char)peek(1)) || ((peek(1) == '+' || peek(1) == '-') && isdigit((unsigned char)peek(2))))) {
        is_float = true;
        i += 2;
        while (isdigit((unsigned char)peek())) i++;
      }
      std::string num = s.substr(b, i - b);
      while (i < s.size() && (isalnum((unsigned char)s[i]) || s[i] == '_')) t.suffix += s[i++];
      if (is_float) {
        t.kind = T::Float;
        t.text = num;
      } else {
        t.kind = T::Int;
        t.ival = strtoull(num.c_str(), nullptr, 10);
      }
      out.push_back(t);
      continue;
    }
    if (c == '-' && peek(1) == '-' && peek(2) == '-') {
      while (peek() == '-') i++;
      t.kind = T::Sep;
      t.text = "---";
      out.push_back(t);
      continue;
    }
    static const char* two[] = {"->", "==", "!=", "<=", ">=", "&&", "||", "<<", ">>"};
    t.kind = T::Punct;
    bool matched = false;
    for (const char* p : two)
      if (c == p[0] && peek(1) == p[1]) {
        t.text = p;
        i += 2;
        matched = true;
        break;
      }
    if (!matched) {
      t.text = std::string(1, c);
      i++;
    }
    out.push_back(t);
  }
  Tok e;
  e.line = line;
  out.push_back(e);
  return out;
}

struct Parser {
  std::vector<Tok> toks;
  size_t p = 0;
  std::set<std::string> type_names;
  Program prog;

  const Tok& cur() const { return toks[p]; }
  const Tok& look(size_t k = 1) const { return toks[std::min(p + k, toks.size() - 1)]; }
  [[noreturn]] void fail(const std::string& what) const {
    throw LayoutError("line " + std::to_string(cur().line) + ": " + what + " (at '" + (cur().kind == T::End ? "<eof>" : cur().kind == T::Int ? std::to_string(cur().ival) : cur().text) + "')");
  }
  bool is_punct(const char* s) const { return cur().kind == T::Punct && cur().text == s; }
  bool is_kw(const char* s) const { return cur().kind == T::Ident && cur().text == s; }
  bool accept(const char* s) {
    if (is_punct(s)) { p++; return true; }
    return false;
  }
  void expect(const char* s) {
    if (!accept(s)) fail(std::string("expected '") + s + "'");
  }
  std::string ident(const char* what = "identifier") {
    if (cur().kind != T::Ident) fail(std::string("expected ") + what);
    return toks[p++].text;
  }

  // ----------------------------------------------------------------- types
  static bool all_digits(const std::string& s, size_t from) {
    if (from >= s.size()) return false;
    for (size_t i = from; i < s.size(); i++)
      if (!isdigit((unsigned char)s[i])) return false;
    return true;
  }
  TypeP type_from_ident(const std::string& id, bool strict) const {
    auto mk = [] { return std::make_shared<Type>(); };
    if (id == "bool") { auto t = mk(); t->kind = Type::Bool; t->width = 1; return t; }
    if (id == "ptr") { auto t = mk(); t->kind = Type::Ptr; t->width = 64; return t; }
    if (id == "f32" || id == "f16") { auto t = mk(); t->kind = Type::Float; t->width = id == "f32" ? 32 : 16; return t; }
    if ((id[0] == 'u' || id[0] == 'i') && all_digits(id, 1)) {
      uint32_t w = (uint32_t)strtoul(id.c_str() + 1, nullptr, 10);
      if (w < 1 || w > 64) return nullptr;
      auto t = mk();
      t->kind = Type::Int;
      t->width = w;
      t->is_signed = id[0] == 'i';
      return t;
    }
    if (type_names.count(id)) { auto t = mk(); t->kind = Type::Named; t->name = id; return t; }
    size_t x = id.rfind('x');
    if (x != std::string::npos && x > 0 && all_digits(id, x + 1)) {
      TypeP base = type_from_ident(id.substr(0, x), true);
      if (base) {
        auto t = mk();
        t->kind = Type::Vec;
        t->elem = base;
        t->lanes = (uint32_t)strtoul(id.c_str() + x + 1, nullptr, 10);
        return t;
      }
    }
    if (strict) return nullptr;
    auto t = mk();
    t->kind = Type::Named;
    t->name = id;
    return t;
  }
  bool ident_is_type(const std::string& id) const { return type_from_ident(id, true) != nullptr; }

  TypeP parse_type() {
    TypeP t;
    if (accept("(")) {
      t = std::make_shared<Type>();
      t->kind = Type::Tuple;
      do t->members.push_back(parse_type()); while (accept(","));
      expect(")");
    } else {
      std::string id = ident("type");
      if ((id == "option" || id == "set") && is_punct("[")) {  // only met in algorithm files
        p++;
        TypeP inner = parse_type();
        expect("]");
        t = std::make_shared<Type>();
        t->kind = Type::Named;
        t->name = id + "[" + inner->str() + "]";
      } else {
        t = type_from_ident(id, false);
        if (!t) fail("bad type '" + id + "'");
      }
    }
    while (is_punct("[")) {
      p++;
      auto a = std::make_shared<Type>();
      a->kind = Type::Array;
      a->elem = t;
      if (cur().kind == T::Int) a->lanes = (uint32_t)toks[p++].ival;
      else a->len_field = ident("array length");
      expect("]");
      t = a;
    }
    return t;
  }

  std::vector<Param> parse_params() {
    std::vector<Param> ps;
    expect("(");
    if (!is_punct(")")) {
      do {
        Param q;
        q.name = ident("parameter name");
        expect(":");
        if (is_kw("mut")) p++;
        q.type = parse_type();
        if (accept("=")) q.default_value = parse_expr();
        ps.push_back(q);
      } while (accept(","));
    }
    expect(")");
    return ps;
  }

  // ----------------------------------------------------------------- expressions
  ExprP mk(Expr::Kind k) {
    auto e = std::make_shared<Expr>();
    e->kind = k;
    e->line = cur().line;
    return e;
  }
  ExprP parse_expr() { return parse_bin(0); }
  int prec_of(const Tok& t) const {
    if (t.kind != T::Punct) return -1;
    static const std::map<std::string, int> pr = {{"||", 1}, {"&&", 2}, {"|", 3}, {"^", 4}, {"&", 5}, {"==", 6}, {"!=", 6}, {"<", 7}, {"<=", 7}, {">", 7}, {">=", 7}, {"<<", 8}, {">>", 8}, {"+", 9}, {"-", 9}, {"*", 10}, {"/", 10}, {"%", 10}};
    auto it = pr.find(t.text);
    return it == pr.end() ? -1 : it->second;
  }
  ExprP parse_bin(int min_prec) {
    ExprP lhs = parse_unary();
    for (;;) {
      int pr = prec_of(cur());
      if (pr < 0 || pr < min_prec) break;
      std::string op = toks[p++].text;
      ExprP rhs = parse_bin(pr + 1);
      auto e = mk(Expr::Binary);
      e->text = op;
      e->args = {lhs, rhs};
      lhs = e;
    }
    return lhs;
  }
  ExprP parse_unary() {
    if (is_punct("-") || is_punct("!") || is_punct("~")) {
      auto e = mk(Expr::Unary);
      e->text = toks[p++].text;
      e->args = {parse_unary()};
      return e;
    }
    return parse_cast();
  }
  ExprP parse_cast() {  // `as` / `to` bind tighter than any binary operator (parser.cpp:467-489)
    ExprP e = parse_postfix();
    while (is_kw("as") || is_kw("to")) {
      auto c = mk(Expr::Cast);
      c->bitcast = toks[p++].text == "to";
      c->type = parse_type();
      c->args = {e};
      e = c;
    }
    return e;
  }
  ExprP parse_postfix() {
    ExprP e = parse_primary();
    for (;;) {
      if (is_punct(".")) {
        p++;
        auto m = mk(Expr::Member);
        if (cur().kind == T::Int) m->text = std::to_string(toks[p++].ival);
        else m->text = ident("member name");
        m->args = {e};
        e = m;
      } else if (is_punct("[")) {
        p++;
        ExprP a = parse_expr();
        if (accept(":")) {
          ExprP b = parse_expr();
          auto r = mk(Expr::Range);
          r->args = {e, a, b};
          e = r;
        } else {
          auto ix = mk(Expr::Index);
          ix->args = {e, a};
          e = ix;
        }
        expect("]");
      } else {
        break;
      }
    }
    return e;
  }
  ExprP parse_primary() {
    const Tok& t = cur();
    if (t.kind == T::Int) {
      auto e = mk(Expr::IntLit);
      e->ival = t.ival;
      e->has_u = !t.suffix.empty();
      p++;
      return e;
    }
    if (t.kind == T::Float) {
      auto e = mk(Expr::FloatLit);
      e->text = t.text;
      p++;
      return e;
    }
    if (is_punct("(")) {
      p++;
      ExprP first = parse_expr();
      if (is_punct(",")) {
        auto tu = mk(Expr::Tuple);
        tu->args.push_back(first);
        while (accept(",")) tu->args.push_back(parse_expr());
        expect(")");
        return tu;
      }
      expect(")");
      return first;
    }
    if (is_punct("{")) {
      p++;
      auto b = mk(Expr::Brace);
      if (!is_punct("}")) do b->args.push_back(parse_expr()); while (accept(","));
      expect("}");
      return b;
    }
    if (in_build && is_kw("build")) {  // `let R: u32 = build right;`
      p++;
      auto e = mk(Expr::BuildChild);
      e->text = ident("child name");
      return e;
    }
    if (t.kind == T::Ident) {
      std::string id = toks[p++].text;
      if (is_punct("{") && ident_is_type(id)) {  // T { a, b, c }
        p++;
        auto c = mk(Expr::Construct);
        c->type = type_from_ident(id, true);
        if (!is_punct("}")) do c->args.push_back(parse_expr()); while (accept(","));
        expect("}");
        return c;
      }
      if (is_punct("(")) {
        p++;
        ExprP c;
        if (ident_is_type(id)) {  // record constructor call syntax: AABB(lo, hi)
          c = mk(Expr::Construct);
          c->type = type_from_ident(id, true);
        } else {
          c = mk(Expr::Call);
          c->text = id;
        }
        if (!is_punct(")")) do c->args.push_back(parse_expr()); while (accept(","));
        expect(")");
        return c;
      }
      auto e = mk(Expr::Ident);
      e->text = id;
      return e;
    }
    fail("expected an expression");
  }

  // ----------------------------------------------------------------- statements
  std::vector<StmtP> parse_block() {
    std::vector<StmtP> out;
    expect("{");
    while (!is_punct("}")) out.push_back(parse_stmt());
    expect("}");
    return out;
  }
  bool in_build = false;  // inside a constructor of a `build` block: `build ...` statements and expressions are legal
  StmtP parse_stmt() {
    auto s = std::make_shared<Stmt>();
    if (in_build && is_kw("build")) {
      p++;
      if (is_kw("root") && look().kind == T::Punct && look().text == "{") {
        p++;
        s->kind = Stmt::BuildRoot;
        s->then_body = parse_block();
        accept(";");
        return s;
      }
      s->kind = Stmt::Build;
      s->name = ident("field or child name");
      if (accept("=")) s->value = parse_expr();
      expect(";");
      return s;
    }
    if (is_kw("let")) {
      p++;
      s->kind = Stmt::Let;
      s->name = ident();
      expect(":");
      if (is_kw("mut")) { p++; s->is_mut = true; }
      s->type = parse_type();
      expect("=");
      s->value = parse_expr();
      expect(";");
      return s;
    }
    if (cur().kind == T::Ident && look().kind == T::Punct && look().text == ":" && !is_kw("return")) {
      s->kind = Stmt::Let;  // `t : mut f32x3 = v;`
      s->name = ident();
      expect(":");
      if (is_kw("mut")) { p++; s->is_mut = true; }
      s->type = parse_type();
      expect("=");
      s->value = parse_expr();
      expect(";");
      return s;
    }
    if (is_kw("if")) {
      p++;
      s->kind = Stmt::If;
      s->cond = parse_expr();
      s->then_body = parse_block();
      if (is_kw("else") || is_kw("elif")) {
        bool elif = toks[p++].text == "elif";
        if (elif || is_kw("if")) {
          if (elif) p--, toks[p].text = "if";
          s->else_body = {parse_stmt()};
        } else {
          s->else_body = parse_block();
        }
      }
      return s;
    }
    if (is_kw("return")) {
      p++;
      s->kind = Stmt::Return;
      if (!is_punct(";")) s->value = parse_expr();
      expect(";");
      return s;
    }
    ExprP e = parse_expr();
    if (accept("=")) {
      s->kind = Stmt::Assign;
      s->lhs = e;
      s->value = parse_expr();
    } else {
      s->kind = Stmt::ExprS;
      s->value = e;
    }
    expect(";");
    return s;
  }

  // ----------------------------------------------------------------- declarations
  void skip_balanced_block() {  // current token is '{'
    int depth = 0;
    do {
      if (cur().kind == T::End) fail("unterminated block");
      if (is_punct("{")) depth++;
      if (is_punct("}")) depth--;
      p++;
    } while (depth > 0);
    accept(";");
  }
  void parse_type_decl() {
    p++;  // type
    TypeDecl d;
    d.name = ident("type name");
    type_names.insert(d.name);
    if (is_punct("(")) d.fields = parse_params();
    if (accept("=")) {
      do {
        Variant v;
        v.name = ident("variant name");
        if (is_punct("(")) v.fields = parse_params();
        d.variants.push_back(v);
      } while (accept("|"));
    }
    accept(";");
    prog.types.push_back(d);
  }
  void parse_func_decl() {
    p++;  // func
    Func f;
    f.name = ident("function name");
    if (is_punct("[")) {  // attribute list, e.g. [recursive]
      while (!is_punct("]")) p++;
      p++;
    }
    f.params = parse_params();
    if (accept("->")) f.ret = parse_type();
    if (is_punct("=")) {  // expression-bodied traversal entry: not layout language — skip it
      while (cur().kind != T::End && !is_kw("func") && !is_kw("type") && !is_kw("layout") && !is_kw("build")) {
        if (is_punct("{")) { skip_balanced_block(); continue; }
        p++;
      }
      return;
    }
    f.body = parse_block();
    prog.funcs.push_back(f);
  }
  Arm parse_arm() {
    Arm a;
    if (is_kw("_")) {
      p++;
      a.pat = Arm::Wildcard;
    } else {
      if (accept(">")) a.pat = Arm::Gt;
      else if (accept("<")) a.pat = Arm::Lt;
      else if (accept(">=")) a.pat = Arm::Ge;
      else if (accept("<=")) a.pat = Arm::Le;
      else a.pat = Arm::Literal;
      bool neg = accept("-");
      if (cur().kind != T::Int) fail("expected a pattern literal");
      a.value = (int64_t)toks[p++].ival;
      if (neg) a.value = -a.value;
    }
    expect("->");
    a.variant = ident("variant name");
    if (is_kw("from")) {
      p++;
      a.is_from = true;
      a.from_group = ident("group name");
      expect("[");
      a.from_key = parse_expr();
      expect("]");
    } else {
      expect("{");
      while (!is_punct("}")) a.members.push_back(parse_member());
      expect("}");
    }
    accept(";");
    return a;
  }
  MemberP parse_member() {
    auto m = std::make_shared<MemberNode>();
    if (cur().kind == T::Sep) {
      p++;
      m->kind = MemberNode::Separator;
      return m;
    }
    if (cur().kind == T::Int) {
      m->kind = MemberNode::Padding;
      m->padding_bits = toks[p++].ival;
      expect(";");
      return m;
    }
    if (is_kw("let")) {
      p++;
      m->kind = MemberNode::Let;
      m->name = ident();
      expect(":");
      m->type = parse_type();
      expect("=");
      m->value = parse_expr();
      expect(";");
      return m;
    }
    if (is_kw("split")) {
      p++;
      m->kind = MemberNode::Split;
      m->value = parse_expr();
      expect("{");
      while (!is_punct("}")) m->arms.push_back(parse_arm());
      expect("}");
      accept(";");
      return m;
    }
    bool indirect = false;
    if (is_kw("indirect")) {
      p++;
      indirect = true;
      if (!is_kw("group")) fail("expected 'group'");
    }
    if (is_kw("group")) {
      p++;
      m->kind = MemberNode::Group;
      m->indirect = indirect;
      if (cur().kind == T::Ident && !is_kw("by")) m->group_name = ident();
      if (accept("[")) {
        do {
          if (cur().kind == T::Int) m->tile = toks[p++].ival;
          else if (is_kw("size")) { p++; expect("="); m->size_expr = parse_expr(); }
          else if (is_kw("align")) {
            p++;
            expect("=");
            if (cur().kind != T::Int) fail("expected an alignment");
            m->align = toks[p++].ival;
            if (m->align == 0 || (m->align & (m->align - 1))) fail("alignment must be a power of two");
          } else fail("expected size, align or a tile count");
        } while (accept(","));
        expect("]");
      }
      if (is_kw("by")) { p++; m->index_binding = ident("index name"); }
      expect("{");
      while (!is_punct("}")) m->members.push_back(parse_member());
      expect("}");
      accept(";");
      return m;
    }
    m->name = ident("member");
    if (accept(":")) {
      m->kind = MemberNode::Stored;
      m->type = parse_type();
      expect(";");
      return m;
    }
    if (accept("=")) {
      m->kind = MemberNode::Derive;
      m->value = parse_expr();
      expect(";");
      return m;
    }
    fail("expected ':' or '='");
  }
  void parse_layout_decl() {
    p++;  // layout
    Layout l;
    l.name = ident("layout name");
    l.ref = parse_params();
    expect("{");
    while (!is_punct("}")) l.members.push_back(parse_member());
    expect("}");
    accept(";");
    prog.layouts.push_back(l);
  }
  void parse_build_decl() {
    p++;  // build
    const std::string adt = ident("build name");
    std::string order = "pre";
    if (accept("[")) {
      if (is_kw("order")) {
        p++;
        expect("=");
        order = ident("pre or post");
        if (order != "pre" && order != "post") fail("invalid build order");
      }
      expect("]");
    }
    prog.build_orders.push_back(order);
    BuildDecl bd;
    bd.adt = adt;
    bd.order = order;
    expect("{");
    while (!is_punct("}")) {
      if (!is_kw("build")) fail("expected 'build Variant(...)'");
      p++;
      BuildCtor c;
      c.variant = ident("variant name");
      expect("(");
      if (!is_punct(")")) do {
        Param pa;
        pa.name = ident("parameter name");
        expect(":");
        pa.type = parse_type();
        c.params.push_back(pa);
      } while (accept(","));
      expect(")");
      in_build = true;
      c.body = parse_block();
      in_build = false;
      accept(";");
      bd.ctors.push_back(std::move(c));
    }
    expect("}");
    accept(";");
    prog.builds.push_back(std::move(bd));
  }
  void run() {
    while (cur().kind != T::End) {
      if (is_kw("type")) parse_type_decl();
      else if (is_kw("func")) parse_func_decl();
      else if (is_kw("layout")) parse_layout_decl();
      else if (is_kw("build")) parse_build_decl();
      else fail("expected 'type', 'func', 'layout' or 'build'");
    }
  }
};

const char* kPrelude = "type Triangle(p0: f32x3, p1: f32x3, p2: f32x3);\n";

}  // namespace

Program parse_program(const std::vector<std::string>& sources) {
  // pre-scan for declared type names so that uses may precede declarations across files
  Parser ps;
  bool has_triangle = false;
  std::string all;
  for (auto& s : sources) {
    all += s;
    all += "\n";
  }
  {
    std::vector<Tok> pre = lex(all);
    for (size_t i = 0; i + 1 < pre.size(); i++)
      if (pre[i].kind == T::Ident && pre[i].text == "type" && pre[i + 1].kind == T::Ident) {
        ps.type_names.insert(pre[i + 1].text);
        if (pre[i + 1].text == "Triangle") has_triangle = true;
      }
  }
  if (!has_triangle) {
    all = std::string(kPrelude) + all;
    ps.type_names.insert("Triangle");
  }
  ps.toks = lex(all);
  ps.run();
  return std::move(ps.prog);
}

}  // namespace scion::lc
