// okt_gen.cpp — seeded synthetic inputs, bit-exact with the reference's
// generators (rounded to fp32):
//   random_dense               proj/tests/test_util.hpp:135-140
//   drifting_gradient_process  proj/core/src/trainer.cpp:338-388
// The O(n) noise runs on the device; the n/100 heavy slots keep the
// reference's sequential linear-probing placement and are computed on the host.
// Not on the hot path: these feed the bench and the GPU parity tests.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/okt.h"
#include "okt_kernels.hpp"

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

uint64_t splitmix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t mix64(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (kGamma + b + (a << 6) + (a >> 2)));
}
double unit_from_bits(uint64_t bits) { return double(bits >> 11) * 0x1.0p-53; }

int launch_ctx(okt::Launch& L, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  L.sms = sms;
  L.s = static_cast<cudaStream_t>(stream);
  return 0;
}

}  // namespace

extern "C" {

int okt_gen_random_dense(float* d_out, size_t n, uint64_t seed, void* stream) {
  okt::Launch L;
  launch_ctx(L, stream);
  cudaError_t e = okt::launch_gen_random_dense(L, d_out, n, seed);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.s);
  return e == cudaSuccess ? OKT_OK : OKT_ERR_CUDA;
}

int okt_gen_drift(float* d_out, size_t n, int64_t t, uint64_t seed, uint64_t rank_key, int fixed_positions,
                  void* stream) {
  if (t < 1) return OKT_ERR_INVALID_ARGUMENT;
  if (n == 0) return OKT_OK;
  okt::Launch L;
  launch_ctx(L, stream);
  const uint64_t epoch = uint64_t((t - 1) / 1024);
  const double scale = std::pow(0.95, double(epoch));
  const uint64_t strm = mix64(seed, mix64(0x72616e6bu, rank_key));
  const uint64_t pair = uint64_t((t + 1) / 2);
  const double noise_sign = (t % 2 == 1) ? 1.0 : -1.0;
  const uint64_t noise_key = mix64(mix64(strm, 0x6e6f6973u), pair);
  // g[i] = noise_sign * 0.04 * scale * (2u - 1), evaluated left to right.
  const double coef = noise_sign * 0.04 * scale;
  cudaError_t e = okt::launch_gen_noise(L, d_out, n, noise_key, coef);
  if (e != cudaSuccess) return OKT_ERR_CUDA;

  const uint64_t heavy_epoch = fixed_positions ? 0 : epoch;
  const uint64_t pos_key = mix64(mix64(seed, 0x65706f73u), heavy_epoch);
  const uint64_t mag_key = mix64(mix64(strm, 0x656d6167u), heavy_epoch);
  const uint64_t jit_key = mix64(strm, 0x6a697474u);
  const size_t slots = std::max<size_t>(1, n / 100);
  std::vector<uint8_t> taken(n, 0);
  std::vector<uint32_t> pos(slots);
  std::vector<float> val(slots);
  for (size_t h = 0; h < slots; ++h) {
    size_t p = size_t(mix64(pos_key, h) % n);
    while (taken[p]) p = (p + 1) % n;
    taken[p] = 1;
    const uint64_t mag_bits = mix64(mag_key, h);
    double mag = (1.0 + unit_from_bits(mag_bits)) * scale;
    if (!fixed_positions) {
      const double u = unit_from_bits(mix64(mix64(jit_key, uint64_t(t)), h));
      mag *= 1.0 + 0.08 * (2.0 * u - 1.0);
    }
    pos[h] = uint32_t(p);
    val[h] = float((mag_bits & 1u) ? mag : -mag);
  }
  uint32_t* d_pos = nullptr;
  float* d_val = nullptr;
  e = cudaMalloc(&d_pos, 4 * slots);
  if (e == cudaSuccess) e = cudaMalloc(&d_val, 4 * slots);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_pos, pos.data(), 4 * slots, cudaMemcpyHostToDevice, L.s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_val, val.data(), 4 * slots, cudaMemcpyHostToDevice, L.s);
  if (e == cudaSuccess) e = okt::launch_scatter_heavy(L, d_pos, d_val, slots, d_out);
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.s);
  cudaFree(d_pos);
  cudaFree(d_val);
  return e == cudaSuccess ? OKT_OK : OKT_ERR_CUDA;
}

}  // extern "C"
