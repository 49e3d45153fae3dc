// harness_main.cpp — command-line entry for the reference's own harness (evomem::run, run.hpp:10-32)
// linked against the GPU adapter instead of attention_tiled.cpp (see integration/Makefile).
//   evomem_gpu_harness <attn-bench|gradcheck|precision-demo> [--config PATH] [--output PATH]
//                      [--format csv|json] [--seed N]
#include <cstdlib>
#include <iostream>
#include <string>

#include "evomem/run.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: " << argv[0] << " <command> [--config PATH] [--output PATH] [--format csv|json] [--seed N]\n";
    return 1;
  }
  evomem::RunSpec spec;
  spec.command = argv[1];
  spec.output_path = "/dev/stdout";
  for (int i = 2; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--config") spec.config_path = v;
    else if (k == "--output") spec.output_path = v;
    else if (k == "--format") spec.format = v == "json" ? evomem::ReportFormat::Json : evomem::ReportFormat::Csv;
    else if (k == "--seed") spec.seed = std::strtoull(v.c_str(), nullptr, 10);
    else {
      std::cerr << "unknown option " << k << "\n";
      return 1;
    }
  }
  return evomem::run(spec, std::cerr);
}
