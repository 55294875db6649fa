// scionc — command-line front door of the layout compiler (the slice of the reference CLI's
// `check` / `footprint` / `compile --emit-c` subcommands, that the B200 backend needs).
//   scionc plan      <registry-name> <file.scion>...   -> MemoryPlan JSON on stdout
//   scionc emit-cuda <registry-name> <file.scion>...   -> CUDA header on stdout
//   scionc stats     <registry-name> <file.scion>...   -> op-count JSON of the decode, per variant (SPEC.md:360 --dump-stats)
//   scionc emit-c    <registry-name> <file.scion>...   -> C11 header: packed node records + static assertions + slot table
// exit codes follow the reference CLI: 0 ok, 1 diagnostics, 2 usage.
#include <fstream>
#include <iostream>
#include <sstream>

#include "../layoutc/layoutc.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::cerr << "usage: scionc {plan|emit-cuda|emit-c|stats} <registry-name> <file.scion>...\n";
    return 2;
  }
  std::string cmd = argv[1], name = argv[2];
  std::vector<std::string> srcs;
  for (int i = 3; i < argc; i++) {
    std::ifstream in(argv[i], std::ios::binary);
    if (!in) {
      std::cerr << "scionc: cannot open " << argv[i] << "\n";
      return 2;
    }
    std::ostringstream os;
    os << in.rdbuf();
    srcs.push_back(os.str());
  }
  try {
    scion::lc::Program prog = scion::lc::parse_program(srcs);
    scion::lc::Plan plan = scion::lc::plan_layout(prog, name);
    if (cmd == "plan") std::cout << plan.to_json() << "\n";
    else if (cmd == "emit-cuda") std::cout << scion::lc::emit_cuda(plan);
    else if (cmd == "emit-c") std::cout << scion::lc::emit_c_records(plan);
    else if (cmd == "stats") std::cout << scion::lc::decode_stats_json(plan) << "\n";
    else {
      std::cerr << "scionc: unknown command " << cmd << "\n";
      return 2;
    }
  } catch (const std::exception& e) {
    std::cerr << "scionc: " << name << ": error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
