// Dispatcher of the persistent cooperative PCG solver.
#include "persist_core.cuh"

namespace ga {

bool persist_launch_p1(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p2(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p3(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p4(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p5(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p6(const PersistArgs& A, cudaStream_t s);
bool persist_launch_p7(const PersistArgs& A, cudaStream_t s);

bool persist_supported(const PersistArgs& A) { return persist_supported_impl(A); }

bool launch_pcg_persist(const PersistArgs& A, cudaStream_t s) {
  switch (A.pa.p) {
    case 1: return persist_launch_p1(A, s);
    case 2: return persist_launch_p2(A, s);
    case 3: return persist_launch_p3(A, s);
    case 4: return persist_launch_p4(A, s);
    case 5: return persist_launch_p5(A, s);
    case 6: return persist_launch_p6(A, s);
    default: return persist_launch_p7(A, s);
  }
}

}  // namespace ga
