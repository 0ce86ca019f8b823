// kernel_oneblock_shapes.cu -- single-block kernel instantiations for the other
// fixed-length shapes of BASELINE.json cfg2 / cfg3: 32-, 64- and 128-byte
// messages for every variant whose rate leaves room for the pad byte, with the
// variant's digest (or 32 / 64 / 128 bytes of SHAKE output).  UNROLL 23 (peeled 1 + 7x3 + 2), ALU only.
#include "oneblock.cuh"

namespace b200sha3 {

// (rate lanes, message lanes, output 32-bit words)
#define B200SHA3_SHAPES(X)                                                   \
  X(18, 4, 7) X(18, 8, 7) X(18, 16, 7)     /* SHA3-224: 32/64/128 B -> 28 B */ \
  X(17, 4, 8) X(17, 16, 8)                 /* SHA3-256 / SHAKE256 -> 32 B    */ \
  X(13, 4, 12) X(13, 8, 12)                /* SHA3-384: 32/64 B -> 48 B      */ \
  X(9, 4, 16) X(9, 8, 16)                  /* SHA3-512: 32/64 B -> 64 B      */ \
  X(21, 4, 8) X(21, 8, 8) X(21, 16, 8)     /* SHAKE128 -> 256 bits           */ \
  X(21, 8, 16) X(21, 8, 32)                /* SHAKE128 64 B -> 512 / 1024 bits */ \
  X(17, 8, 16) X(17, 8, 32)                /* SHAKE256 64 B -> 512 / 1024 bits */

bool oneblock_shape_exists(int rl, int ml, int ow) {
  if (rl == 17 && ml == 8 && ow == 8) return true;  // the tuning-matrix shape
#define X(RL, ML, OW) \
  if (rl == RL && ml == ML && ow == OW) return true;
  B200SHA3_SHAPES(X)
#undef X
  return false;
}

cudaError_t launch_oneblock_shape(int rl, int ml, int ow, const HashArgs& args,
                                  const LaunchPlan& plan, cudaStream_t stream) {
#define X(RL, ML, OW)                      \
  if (rl == RL && ml == ML && ow == OW)    \
    return launch_oneblock_instance<RL, ML, OW, 23, 0>(args, plan, stream);
  B200SHA3_SHAPES(X)
#undef X
  return cudaErrorNotSupported;
}

}  // namespace b200sha3
