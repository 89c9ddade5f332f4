// complex64 instantiation of the single-gate pass kernels (see kernels.cuh).
#include "kernels.cuh"
namespace qj {
QJ_INSTANTIATE(float)
}
