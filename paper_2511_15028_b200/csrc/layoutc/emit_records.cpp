// emit_records — typed, packed node-record declarations for a planned layout.
//
// SPEC.md:396-404 (emit_c): "packed record declarations matching MemoryPlan strides bit-for-bit ... a static
// assertion on node size"; PAPER Appendix E shows the idiom (`__attribute__((packed))`).  One struct per buffer
// segment: stored fields in slot order with their C types (bit-fields where a field is not byte-granular — GCC / Clang /
// NVCC pack bit-fields LSB first and, in a packed struct, across storage-unit boundaries, which is the little-endian
// LSB-first convention of /root/reference/proj/src/bits.cpp:7-36), split arms as an anonymous union of anonymous
// structs (arms overlay the widest arm, plan.cpp:174-241), explicit padding up to the planned stride, and static
// assertions on the size and on the byte offset of every byte-granular field.  The same text serves the CUDA header
// (emit_cuda) and the C11 header of `scionc emit-c`; the decode routines do not go through these structs (they extract
// from vector-loaded words), the structs are the layout's ABI for anything that wants to read or write a record by
// field, and tests/test_layoutc.py checks that a record written through them decodes to the same values.
#include <algorithm>
#include <functional>
#include <sstream>

#include "layoutc.hpp"

namespace scion::lc {
namespace {

struct Item {
  const Slot* slot;
  const MemberNode* split = nullptr;  // outermost split the field sits in (null: common to all variants)
  int arm = -1;
};

struct RecordEmitter {
  const Plan& plan;
  const Program& prog;
  bool c11;
  std::ostringstream out;
  int pad_id = 0;
  std::vector<std::pair<std::string, uint64_t>> byte_members;  // (member path, byte offset) for the offsetof assertions

  RecordEmitter(const Plan& p, bool c) : plan(p), prog(*p.program), c11(c) {}

  static bool whole(uint32_t w) { return w == 8 || w == 16 || w == 32 || w == 64; }
  // every scalar leaf of the type is 8/16/32/64 bits wide (=> representable without bit-fields at a byte boundary)
  bool byte_typed(const TypeP& t) const {
    switch (t->kind) {
      case Type::Int: return whole(t->width);
      case Type::Float: return true;
      case Type::Ptr: return true;
      case Type::Bool: return false;
      case Type::Vec: case Type::Array: return t->len_field.empty() && byte_typed(t->elem);
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        if (!d || d->is_adt()) return false;
        for (auto& f : d->fields)
          if (!byte_typed(f.type)) return false;
        return true;
      }
      case Type::Tuple: return false;
    }
    return false;
  }
  std::string scalar(const TypeP& t) const {
    if (t->kind == Type::Float) return "float";
    if (t->kind == Type::Ptr) return "uint64_t";
    return std::string(t->is_signed ? "int" : "uint") + std::to_string(t->width) + "_t";
  }
  // declaration of a byte-typed value: "<type> name<dims>;" (records become anonymous structs)
  void typed_decl(const TypeP& t, const std::string& name, const std::string& dims, int ind) {
    std::string pad((size_t)ind * 2, ' ');
    switch (t->kind) {
      case Type::Vec: case Type::Array: typed_decl(t->elem, name, dims + "[" + std::to_string(t->lanes) + "]", ind); return;
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        out << pad << "struct {  /* " << t->name << " */\n";
        for (auto& f : d->fields) typed_decl(f.type, f.name, "", ind + 1);
        out << pad << "} " << name << dims << ";\n";
        return;
      }
      default: out << pad << scalar(t) << " " << name << dims << ";\n"; return;
    }
  }
  // bit-field form: one bit-field per scalar leaf, names suffixed with the lane / field path
  void bit_decl(const TypeP& t, const std::string& name, int ind) {
    std::string pad((size_t)ind * 2, ' ');
    switch (t->kind) {
      case Type::Vec: case Type::Array:
        for (uint32_t i = 0; i < t->lanes; i++) bit_decl(t->elem, name + "_" + std::to_string(i), ind);
        return;
      case Type::Named: {
        const TypeDecl* d = prog.find_type(t->name);
        for (auto& f : d->fields) bit_decl(f.type, name + "_" + f.name, ind);
        return;
      }
      case Type::Bool: out << pad << "uint8_t " << name << " : 1;\n"; return;
      case Type::Float: out << pad << "uint32_t " << name << " : 32;  /* f32 bits */\n"; return;
      case Type::Ptr: out << pad << "uint64_t " << name << " : 64;\n"; return;
      default: {
        const char* base = t->width <= 8 ? "uint8_t" : t->width <= 16 ? "uint16_t" : t->width <= 32 ? "uint32_t" : "uint64_t";
        out << pad << base << " " << name << " : " << t->width << ";" << (t->is_signed ? "  /* two's complement */" : "") << "\n";
        return;
      }
    }
  }
  void padding(uint64_t& pos, uint64_t to, int ind) {
    if (to <= pos) return;
    std::string pad((size_t)ind * 2, ' ');
    uint64_t gap = to - pos;
    if (pos % 8 == 0 && gap % 8 == 0) {
      out << pad << "uint8_t pad" << pad_id++ << "_[" << gap / 8 << "];\n";
    } else {
      while (gap > 0) {
        const uint64_t w = gap > 32 ? 32 : gap;
        out << pad << "uint32_t : " << w << ";\n";
        gap -= w;
      }
    }
    pos = to;
  }
  // one stored field at its planned offset; `prefix` = path of the enclosing anonymous aggregates (empty: they are anonymous)
  void field(const Slot& s, uint64_t& pos, int ind, bool record_offsets) {
    padding(pos, s.offset, ind);
    if (s.offset % 8 == 0 && s.width % 8 == 0 && byte_typed(s.type)) {
      typed_decl(s.type, s.name, "", ind);
      if (record_offsets) byte_members.push_back({s.name, s.offset / 8});
    } else {
      bit_decl(s.type, s.name, ind);
    }
    pos = s.offset + s.width;
  }

  void record(const Buffer& b, size_t seg, const std::string& rname) {
    // fields of this segment, each with the outermost split arm it belongs to
    std::vector<Item> items;
    for (auto& s : plan.slots)
      if (s.buffer == b.id && (size_t)s.segment == seg) items.push_back(Item{&s});
    std::function<void(const std::vector<MemberP>&, const MemberNode*, int)> walk = [&](const std::vector<MemberP>& ms, const MemberNode* split, int arm) {
      for (auto& m : ms) {
        if (m->kind == MemberNode::Stored)
          for (auto& it : items)
            if (it.slot->member == m.get()) { it.split = split; it.arm = arm; }
        if (m->kind == MemberNode::Split)
          for (size_t a = 0; a < m->arms.size(); a++) walk(m->arms[a].members, split ? split : m.get(), split ? arm : (int)a);
        if (m->kind == MemberNode::Group) walk(m->members, split, arm);
      }
    };
    walk(plan.layout->members, nullptr, -1);
    std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) { return x.slot->offset < y.slot->offset; });

    out << "struct __attribute__((packed)) " << rname << " {\n";
    uint64_t pos = 0;
    std::set<const MemberNode*> done;
    for (auto& it : items) {
      if (!it.split) {
        field(*it.slot, pos, 1, true);
        continue;
      }
      if (done.count(it.split)) continue;
      done.insert(it.split);
      // the overlay region of this split: every arm starts at the region's first bit
      uint64_t lo = ~0ull, hi = 0;
      int narms = 0;
      for (auto& j : items)
        if (j.split == it.split) { lo = std::min(lo, j.slot->offset); hi = std::max(hi, j.slot->offset + j.slot->width); narms = std::max(narms, j.arm + 1); }
      padding(pos, lo, 1);
      const bool whole_bytes = lo % 8 == 0 && hi % 8 == 0;
      if (whole_bytes) {
        out << "  union {  /* split arms overlay the widest arm */\n";
        for (int a = 0; a < narms; a++) {
          bool any = false;
          for (auto& j : items) any = any || (j.split == it.split && j.arm == a);
          if (!any) continue;
          out << "    struct __attribute__((packed)) {  /* arm " << a << ": " << it.split->arms[(size_t)a].variant << " */\n";
          uint64_t p2 = lo;
          for (auto& j : items)
            if (j.split == it.split && j.arm == a) field(*j.slot, p2, 3, true);
          padding(p2, hi, 3);
          out << "    };\n";
        }
        out << "  };\n";
      } else {
        // sub-byte overlay (pbrt-q16: u28 child offset | u28 primitive offset behind a u4 count): C cannot start a union inside a
        // byte, so the shared bits are declared once, named after the first arm's field(s); the arms reinterpret them
        out << "  /* split arms overlay these bits:";
        for (auto& j : items)
          if (j.split == it.split) out << " " << j.slot->name << "@" << j.slot->offset << ":" << j.slot->width << " (" << it.split->arms[(size_t)j.arm].variant << ")";
        out << " */\n";
        uint64_t p2 = lo;
        int first_arm = -1;
        for (auto& j : items)
          if (j.split == it.split && (first_arm < 0 || j.arm == first_arm)) { first_arm = j.arm; field(*j.slot, p2, 1, false); }
        padding(p2, hi, 1);
      }
      pos = hi;
    }
    padding(pos, b.segments[seg].stride_bytes * 8, 1);
    out << "};\n";
    const char* sa = c11 ? "_Static_assert" : "static_assert";
    out << sa << "(sizeof(" << (c11 ? "struct " : "") << rname << ") == " << b.segments[seg].stride_bytes << ", \"node record must match the planned stride\");\n";
    for (auto& [name, off] : byte_members)
      out << sa << "(offsetof(" << (c11 ? "struct " : "") << rname << ", " << name << ") == " << off << ", \"" << name << " must sit at its planned byte offset\");\n";
    byte_members.clear();
  }
};

}  // namespace

// typed packed record declarations of every node buffer of the plan (one struct per segment), named
// `<prefix><buffer>_s<segment>`; c11 selects _Static_assert / `struct` tags
std::string emit_records(const Plan& plan, const std::string& prefix, bool c11) {
  RecordEmitter e(plan, c11);
  for (auto& b : plan.buffers) {
    if (b.segments.empty()) continue;
    for (size_t s = 0; s < b.segments.size(); s++) {
      if (b.is_global_array) {  // the primitive array: elements are opaque to the layout (Triangle = 9 x f32)
        e.out << "struct __attribute__((packed)) " << prefix << ident_of(b.name) << "_s" << s << " { uint8_t bytes[" << b.segments[s].stride_bytes << "]; };\n";
        continue;
      }
      e.record(b, s, prefix + ident_of(b.name) + "_s" + std::to_string(s));
    }
  }
  return e.out.str();
}

// `scionc emit-c`: a self-contained C11 header with the packed record declarations, their static assertions and the
// slot table (buffer, segment, bit offset, width) of the layout — the record half of the reference's emit_c contract
// (SPEC.md:396-404).  The traversal half is the CUDA backend (emit_cuda + device/traverse.cuh): this backend ships no CPU
// execution path.
std::string emit_c_records(const Plan& plan) {
  std::ostringstream out;
  const std::string id = ident_of(plan.layout_name);
  out << "/* GENERATED by scionc emit-c from layout '" << plan.layout_name << "' — do not edit. */\n";
  out << "#ifndef SCION_RECORDS_" << id << "_H\n#define SCION_RECORDS_" << id << "_H\n#include <stddef.h>\n#include <stdint.h>\n\n";
  out << emit_records(plan, "scion_" + id + "_", true);
  out << "\n/* slot table: every stored field of the plan */\nstruct scion_" << id << "_slot { const char* name; int buffer, segment; uint32_t bit_offset, bit_width; };\n";
  out << "static const struct scion_" << id << "_slot scion_" << id << "_slots[] = {\n";
  for (auto& s : plan.slots) out << "  {\"" << s.name << "\", " << s.buffer << ", " << s.segment << ", " << s.offset << "u, " << s.width << "u},\n";
  out << "};\n";
  for (auto& b : plan.buffers) out << "#define SCION_" << id << "_STRIDE_" << ident_of(b.name) << " " << b.node_stride() << "u\n";
  out << "#endif\n";
  return out.str();
}

}  // namespace scion::lc
