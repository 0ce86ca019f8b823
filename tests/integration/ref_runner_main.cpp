// tests/integration/ref_runner_main.cpp -- the drop-in claim, demonstrated: the
// reference's OWN benchmark runner and report writer (proj/tools/sha3cli/runner.cpp,
// report.cpp, workload.cpp -- compiled unmodified from /root/reference) linked against
// our sha3::hash_batch (paper_1902_05320_b200/host/b200sha3_dropin.cpp built with
// -DB200SHA3_USE_REFERENCE_TYPES) instead of the reference's core/src/batch.cpp.
// run_benchmark (runner.cpp:30-76) then drives the GPU engine without knowing it.
//
// Also cross-checks every digest of one batch against the reference's one-shot
// sha3_digest (src/sha3.cpp:60-72), which is still the reference's CPU code.
//
//   ref_runner_on_b200                    the sweep + cross-check above
//   ref_runner_on_b200 vectors F.rsp ...  response files read by the reference's own
//       parser (vectors.cpp, unmodified) and hashed as one batch each by the drop-in
#include <cstdio>
#include <iostream>
#include <string>

#include "report.hpp"
#include "runner.hpp"
#include "sha3/batch.hpp"
#include "sha3/sha3.hpp"
#include "vectors.hpp"
#include "workload.hpp"

namespace {

int verify_files(int argc, char** argv) {
  int status = 0;
  for (int i = 2; i < argc; ++i) {
    const auto algorithm = sha3::bench::algorithm_from_filename(argv[i]);
    if (!algorithm) return 2;
    const sha3::bench::VectorFile file = sha3::bench::load_vector_file(argv[i]);
    sha3::HashBatch batch;
    batch.algorithm = *algorithm;
    if (sha3::variant_info(*algorithm).is_xof()) {
      batch.xof_output_bits = file.output_bits ? file.output_bits : file.entries.at(0).expected.size() * 8;
    }
    for (const auto& e : file.entries) batch.messages.push_back(e.message);
    const sha3::BatchResult res = sha3::hash_batch(batch, {});
    std::size_t ok = 0;
    for (std::size_t k = 0; k < file.entries.size(); ++k) ok += res.digests[k] == file.entries[k].expected;
    std::printf("%s: %zu/%zu\n", argv[i], ok, file.entries.size());
    if (ok != file.entries.size()) status = 1;
  }
  return status;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "vectors") return verify_files(argc, argv);
  sha3::bench::WorkloadSpec spec;
  spec.message_size = 64;
  spec.total_sizes = {64 * 1000, 64 * 100000, 64ull << 20};
  const auto records = sha3::bench::run_benchmark(spec, sha3::EngineConfig{}, 3);
  std::cout << sha3::bench::emit_csv(records);

  const sha3::HashBatch batch = sha3::bench::generate_workload(spec, 64 * 5000);
  const sha3::BatchResult res = sha3::hash_batch(batch, {});
  std::size_t bad = 0;
  for (std::size_t i = 0; i < batch.messages.size(); ++i) {
    bad += res.digests[i] != sha3::sha3_digest(batch.algorithm, batch.messages[i]);
  }
  std::printf("cross-check: %zu/%zu digests equal the reference's sha3_digest\n",
              batch.messages.size() - bad, batch.messages.size());
  return bad == 0 ? 0 : 1;
}
