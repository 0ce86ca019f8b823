// version.cu -- b200sha3_version(): version + build provenance.  Compiled by the LINK rule of the
// Makefile (not with the other objects), so the time in the string is the time the library was
// linked: a round summary can tell a library rebuilt on the GPU box from one shipped with the tree.
#include "../../include/b200sha3.h"

#define B200SHA3_STR2(x) #x
#define B200SHA3_STR(x) B200SHA3_STR2(x)

extern "C" const char* b200sha3_version(void) {
  return "b200sha3 0.2 (sm_100a; nvcc " B200SHA3_STR(__CUDACC_VER_MAJOR__) "." B200SHA3_STR(
      __CUDACC_VER_MINOR__) "." B200SHA3_STR(__CUDACC_VER_BUILD__) "; built " __DATE__ " " __TIME__ ")";
}
