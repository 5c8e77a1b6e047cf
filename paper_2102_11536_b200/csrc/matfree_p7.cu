// Instantiation of the matrix-free operator for degree p = 7 (split per p so
// the translation units compile in parallel).
#include "matfree_launch.cuh"

namespace ga {
template void mf_launch_p<7>(const SpmvArgs& a, cudaStream_t s);
}  // namespace ga
