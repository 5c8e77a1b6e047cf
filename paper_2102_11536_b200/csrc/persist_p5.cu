// Instantiation of the persistent PCG solver for degree p = 5 (split per p
// so the translation units compile in parallel).
#include "persist_core.cuh"

namespace ga {

bool persist_launch_p5(const PersistArgs& A, cudaStream_t s) {
  switch (A.pa.kk) {
    case 1: return persist_launch_t<5, 1>(A, s);
    case 2: return persist_launch_t<5, 2>(A, s);
    case 3: return persist_launch_t<5, 3>(A, s);
    default: return persist_launch_t<5, 4>(A, s);
  }
}

}  // namespace ga
