// Open-world layouts (VERDICT r1 missing 6; "constructor specialisation", §7): a layout the
// library was not built with is compiled AT RUN TIME into a plugin and registered under its name —
//   .scion text --parse/check/plan--> Plan --emit_cuda--> gen/<ident>.cuh (decode, records, constructors)
//     --nvcc (device/inst.cu.in: every traversal kernel instantiated for it, same flags as the library)
//     --g++  (host/build_inst.cpp.in: its generated constructors, -frounding-math)
//     --> libscion_layout_<ident>.so --dlopen--> kernel + builder tables
// after which scion_encode (through the layout's own build block), scion_dtree_upload, scion_closest_hit,
// scion_closest_point, scion_collision_detection, scion_ptree_from_buffers ... work for that name like for a built-in.
// Needs nvcc and the library's device sources at run time (SCION_B200_SRC, default: csrc/ next to the library).
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <deque>
#include <fstream>
#include <mutex>
#include <sstream>
#include <stdexcept>

#include "../device/launch.cuh"
#include "build_ctx.hpp"
#include "physical.hpp"

namespace scion {

extern const char* const kBuildNvccFlags;  // build/build_flags.cpp (the Makefile's NVFLAGS / CXXFLAGS, verbatim)
extern const char* const kBuildCxxFlags;

namespace {
struct Dyn {
  std::mutex mu;
  std::deque<LayoutEntry> layouts;      // deque: registered entries never move
  std::deque<std::string> names;        // storage of the C strings the tables point at
  std::deque<KernelEntry> kernels;
  std::deque<BuilderEntry> builders;
};
Dyn& dyn() {
  static Dyn d;
  return d;
}
std::string library_dir() {
  Dl_info info;
  if (dladdr((const void*)&library_dir, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t s = p.rfind('/');
    return s == std::string::npos ? std::string(".") : p.substr(0, s);
  }
  return ".";
}
std::string library_path() {
  Dl_info info;
  if (dladdr((const void*)&library_dir, &info) && info.dli_fname) return info.dli_fname;
  return "libscion_b200.so";
}
bool exists(const std::string& p) {
  struct stat st;
  return ::stat(p.c_str(), &st) == 0;
}
void write_file(const std::string& p, const std::string& s) {
  std::ofstream f(p);
  if (!f) throw std::runtime_error("cannot write " + p);
  f << s;
}
std::string read_file(const std::string& p) {
  std::ifstream f(p);
  if (!f) throw std::runtime_error("cannot read " + p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
std::string replace_all(std::string s, const std::string& a, const std::string& b) {
  for (size_t p = 0; (p = s.find(a, p)) != std::string::npos; p += b.size()) s.replace(p, a.size(), b);
  return s;
}
// runs `cmd`, appends its output to `log`; throws with the tail of the output on failure
void run(const std::string& cmd, std::string& log) {
  log += "$ " + cmd + "\n";
  FILE* p = popen((cmd + " 2>&1").c_str(), "r");
  if (!p) throw std::runtime_error("cannot start: " + cmd);
  char buf[4096];
  std::string out;
  while (size_t n = fread(buf, 1, sizeof buf, p)) out.append(buf, n);
  const int rc = pclose(p);
  log += out;
  if (rc != 0) throw std::runtime_error("layout plugin build step failed (" + cmd.substr(0, cmd.find(' ')) + "): " + (out.size() > 1500 ? out.substr(out.size() - 1500) : out));
}
}  // namespace

const LayoutEntry* dyn_find_layout(const std::string& name) {
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  for (auto& e : d.layouts)
    if (e.name == name) return &e;
  return nullptr;
}
int dyn_layout_count() {
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  return (int)d.layouts.size();
}
const LayoutEntry* dyn_layout_at(int i) {
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  return i >= 0 && i < (int)d.layouts.size() ? &d.layouts[(size_t)i] : nullptr;
}
const KernelEntry* dyn_find_kernels(const char* layout) {
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  for (auto& k : d.kernels)
    if (std::string(k.layout) == layout) return &k;
  return nullptr;
}
const BuilderEntry* dyn_find_builder(const char* layout) {
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  for (auto& k : d.builders)
    if (std::string(k.layout) == layout) return &k;
  return nullptr;
}

// throws std::runtime_error / lc::LayoutError; `log` receives the commands and the compilers' output
void register_layout_plugin(const std::string& name, const std::string& source, const std::string& work_dir_in, std::string& log) {
  static std::mutex registration;  // registrations are serialised: the name check and the table updates belong together
  std::lock_guard<std::mutex> one_at_a_time(registration);
  if (name.empty()) throw std::runtime_error("empty layout name");
  for (char c : name)
    if (!(isalnum((unsigned char)c) || c == '-' || c == '_')) throw std::runtime_error("layout names are [A-Za-z0-9_-]+");
  if (find_layout(name)) throw std::runtime_error("layout '" + name + "' is already registered");
  // 1. front end (throws with the reference's diagnostic classes on ill-formed layouts)
  LayoutEntry e;
  e.name = name;
  e.source = source;
  e.program = std::make_unique<lc::Program>(lc::parse_program({source}));
  e.plan = std::make_unique<lc::Plan>(lc::plan_layout(*e.program, name));
  e.has_cpq = e.plan->family != lc::Family::Bvh8;
  const std::string header = lc::emit_cuda(*e.plan);
  const std::string ident = lc::ident_of(name);
  // 2. sources
  const char* src_env = getenv("SCION_B200_SRC");
  const std::string csrc = src_env && *src_env ? std::string(src_env) : library_dir() + "/csrc";
  if (!exists(csrc + "/device/inst.cu.in") || !exists(csrc + "/host/build_inst.cpp.in"))
    throw std::runtime_error("layout plugins need the library's device sources: " + csrc + "/device/inst.cu.in not found (set SCION_B200_SRC)");
  const char* nvcc_env = getenv("SCION_NVCC");
  const std::string nvcc = nvcc_env && *nvcc_env ? std::string(nvcc_env) : "/usr/local/cuda/bin/nvcc";
  if (!exists(nvcc)) throw std::runtime_error("layout plugins need nvcc at run time: " + nvcc + " not found (set SCION_NVCC)");
  std::string work = work_dir_in;
  if (work.empty()) {
    std::string tmpl = std::string(getenv("TMPDIR") ? getenv("TMPDIR") : "/tmp") + "/scion_layout_XXXXXX";
    if (!mkdtemp(tmpl.data())) throw std::runtime_error("cannot create a work directory under " + tmpl);
    work = tmpl;
  }
  ::mkdir(work.c_str(), 0755);
  ::mkdir((work + "/gen").c_str(), 0755);
  ::mkdir((work + "/build").c_str(), 0755);
  // the stamped units include "../gen/<ident>.cuh", "../device/...", "../host/...": mirror that shape with links
  for (const char* sub : {"device", "host", "layoutc"}) {
    const std::string link = work + "/" + sub;
    ::unlink(link.c_str());
    if (::symlink((csrc + "/" + sub).c_str(), link.c_str()) != 0) throw std::runtime_error("cannot link " + link);
  }
  write_file(work + "/gen/" + ident + ".cuh", header);
  auto stamp = [&](const std::string& in) { return replace_all(replace_all(read_file(in), "@IDENT@", ident), "@NAME@", name); };
  write_file(work + "/build/inst_" + ident + ".cu", stamp(csrc + "/device/inst.cu.in"));
  write_file(work + "/build/build_" + ident + ".cpp", stamp(csrc + "/host/build_inst.cpp.in"));
  write_file(work + "/build/entry_" + ident + ".cpp",
             "#include \"../device/launch.cuh\"\n#include \"../host/build_ctx.hpp\"\nnamespace scion { extern const KernelEntry kKernels_" + ident + "; extern const BuilderEntry kBuilder_" + ident +
                 "; }\nextern \"C\" const void* scion_plugin_kernels() { return &scion::kKernels_" + ident + "; }\nextern \"C\" const void* scion_plugin_builder() { return &scion::kBuilder_" + ident + "; }\n");
  // 3. compile + link: the library's own flags (include paths re-rooted at the work directory and the library's headers)
  const std::string inc = " -I" + work + " -I" + csrc + " -I" + csrc + "/../../include";
  // the plugin is keyed by everything it was compiled from: the emitted header (= layout text + compiler), the two stamped
  // templates, the flags and the library it links against — a caller that passes the same work_dir again reuses it
  uint64_t key = 1469598103934665603ull;  // FNV-1a
  auto mix = [&](const std::string& t) { for (unsigned char c : t) { key ^= c; key *= 1099511628211ull; } };
  mix(header); mix(read_file(csrc + "/device/inst.cu.in")); mix(read_file(csrc + "/host/build_inst.cpp.in")); mix(kBuildNvccFlags); mix(kBuildCxxFlags); mix(name);
  {
    struct stat st;
    if (::stat(library_path().c_str(), &st) == 0) mix(std::to_string((long long)st.st_size) + ":" + std::to_string((long long)st.st_mtime));
  }
  char keyhex[32];
  snprintf(keyhex, sizeof keyhex, "%016llx", (unsigned long long)key);
  const std::string so = work + "/libscion_layout_" + ident + "." + keyhex + ".so";
  if (exists(so)) {
    log += "reusing " + so + "\n";
  } else {
  run("cd " + work + "/build && " + nvcc + " " + kBuildNvccFlags + inc + " -c inst_" + ident + ".cu -o inst_" + ident + ".o", log);
  run("cd " + work + "/build && " + nvcc + " " + kBuildNvccFlags + inc + " -x cu -c entry_" + ident + ".cpp -o entry_" + ident + ".o", log);
  run("cd " + work + "/build && /usr/bin/g++ " + kBuildCxxFlags + inc + " -frounding-math -c build_" + ident + ".cpp -o build_" + ident + ".o", log);
  run("cd " + work + "/build && " + nvcc + " -shared -o " + so + " inst_" + ident + ".o entry_" + ident + ".o build_" + ident + ".o " + library_path() +
          " -Xcompiler -fopenmp -lgomp -ldl -cudart shared",
      log);
  }
  // 4. load + register
  void* h = dlopen(so.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!h) throw std::runtime_error(std::string("cannot load the layout plugin: ") + dlerror());
  auto kern = (const void* (*)())dlsym(h, "scion_plugin_kernels");
  auto bld = (const void* (*)())dlsym(h, "scion_plugin_builder");
  if (!kern || !bld) throw std::runtime_error("layout plugin lacks its entry points");
  Dyn& d = dyn();
  std::lock_guard<std::mutex> lock(d.mu);
  d.names.push_back(name);
  KernelEntry k = *(const KernelEntry*)kern();
  k.layout = d.names.back().c_str();
  BuilderEntry b = *(const BuilderEntry*)bld();
  b.layout = d.names.back().c_str();
  d.kernels.push_back(k);
  d.builders.push_back(b);
  d.layouts.push_back(std::move(e));
}

}  // namespace scion
