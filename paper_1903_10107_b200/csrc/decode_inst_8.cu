// decode_inst_8.cu -- explicit instantiations of decode_kernel (decode_kernel.cuh) launched by kernel_of() in
// qkd_ldpc.cu; the variants are spread over several translation units so nvcc compiles them in parallel.
#include "decode_kernel.cuh"

namespace qkd {

template __global__ void decode_kernel<8, true, true, false, false>(const DecParams);
template __global__ void decode_kernel<8, true, false, false, false>(const DecParams);
template __global__ void decode_kernel<8, true, true, false, true>(const DecParams);
template __global__ void decode_kernel<8, true, false, false, true>(const DecParams);
template __global__ void decode_kernel<8, false, false, false, false>(const DecParams);
template __global__ void decode_kernel<8, false, true, false, false>(const DecParams);

}  // namespace qkd
