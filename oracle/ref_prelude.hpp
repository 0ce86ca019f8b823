// oracle/ref_prelude.hpp -- force-included (-include) when oracle/Makefile
// compiles the reference's core/src/batch.cpp where it lies.
//
// TEST INFRASTRUCTURE ONLY (see oracle/keccak_oracle.c header).
//
// The reference's batch.cpp:108 calls `hash_one(batch, batch.messages[i])`, a
// function that is declared nowhere in the tree, so the file does not compile
// as shipped.  Declaring it here (and defining it in ref_shim.cpp on top of the
// reference's own one-shot functions) lets the UNMODIFIED source compile; no
// reference file is copied or patched.
#pragma once
#include <cstdint>
#include <vector>

namespace sha3 {
struct HashBatch;
std::vector<std::uint8_t> hash_one(const HashBatch& batch,
                                   const std::vector<std::uint8_t>& message);
}  // namespace sha3
