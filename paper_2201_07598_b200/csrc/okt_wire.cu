// okt_wire.cu — the reference's COO wire codec (proj/core/src/sparse.cpp:
// 275-312) on the device: [nnz u32][indices u32 * nnz][values f32 * nnz],
// little endian (the GPU's own byte order), so the image is three u32 arrays
// back to back and both directions are coalesced streaming passes.  Encode
// rounds each fp64 value to fp32 (round to nearest, as static_cast<float>);
// decode validates every index (< n, strictly increasing) in the same pass.
#include "okt_device.cuh"
#include "okt_kernels.hpp"

namespace okt {

__global__ void __launch_bounds__(kThreads)
    wire_encode_kernel(const uint32_t* __restrict__ idx, const double* __restrict__ val, uint64_t nnz,
                       uint32_t* __restrict__ out) {
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = uint32_t(nnz);
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < nnz; i += stride) {
    out[1 + i] = idx[i];
    out[1 + nnz + i] = __float_as_uint(__double2float_rn(val[i]));
  }
}

// bit 0 of *err: an index >= n or not above its predecessor (DecodeError)
__global__ void __launch_bounds__(kThreads)
    wire_decode_kernel(const uint32_t* __restrict__ in, uint64_t nnz, uint64_t n, uint32_t* __restrict__ idx,
                       double* __restrict__ val, uint32_t* err) {
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  bool bad = false;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < nnz; i += stride) {
    const uint32_t v = in[1 + i];
    bad |= v >= n || (i > 0 && v <= in[i]);
    idx[i] = v;
    val[i] = double(__uint_as_float(in[1 + nnz + i]));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1u);
}

cudaError_t launch_wire_encode(Launch& L, const uint32_t* idx, const double* val, uint64_t nnz, uint32_t* out) {
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>((nnz + kThreads - 1) / kThreads, uint64_t(L.sms) * 8)));
  wire_encode_kernel<<<grid, kThreads, 0, L.s>>>(idx, val, nnz, out);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_wire_decode(Launch& L, const uint32_t* in, uint64_t nnz, uint64_t n, uint32_t* idx, double* val,
                               uint32_t* err) {
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>((nnz + kThreads - 1) / kThreads, uint64_t(L.sms) * 8)));
  wire_decode_kernel<<<grid, kThreads, 0, L.s>>>(in, nnz, n, idx, val, err);
  ++L.launches;
  return cudaGetLastError();
}

}  // namespace okt
