// Device copies of the reference RNG (include/gridgnn/rng.hpp:10-76),
// bit-identical 64-bit integer arithmetic.
#pragma once
#include <cstdint>

namespace ggb {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (kGolden + (b << 6) + (b >> 2)));
}

/// The k-th (0-based) next_u64() of Stream(seed) when no earlier call was a
/// rejection: the state advances by kGolden per call (rng.hpp:26-32).
__host__ __device__ __forceinline__ uint64_t stream_draw(uint64_t seed, uint64_t k) {
  return splitmix64(seed + k * kGolden);
}

/// element_unit(key, i, j) >= rate, evaluated exactly on the 53-bit integer:
/// (h >> 11) * 2^-53 >= rate  <=>  (h >> 11) >= thresh, thresh = ceil(rate * 2^53).
__host__ __device__ __forceinline__ bool element_keep(uint64_t row_key, uint64_t j, uint64_t thresh) {
  const uint64_t h = splitmix64(hash_combine(row_key, j));
  return (h >> 11) >= thresh;
}

/// The column term of hash_combine(row_key, j): hash_combine(a, j) =
/// splitmix64(a ^ column_term(j)), so a row kernel computes it once per column.
__host__ __device__ __forceinline__ uint64_t column_term(uint64_t j) { return kGolden + (j << 6) + (j >> 2); }

#ifdef __CUDACC__
/// element_keep(row_key, j, thresh) with cj = column_term(j) and
/// T = thresh << 11 ((h >> 11) >= thresh <=> h >= T for thresh < 2^53): the
/// last multiply of the second splitmix64 is formed for its high word only,
/// and the full hash is finished only when the high words tie (p = 2^-32).
__device__ __forceinline__ bool element_keep_cj(uint64_t row_key, uint64_t cj, uint64_t T) {
  const uint64_t h1 = splitmix64(row_key ^ cj);
  uint64_t x = h1 + kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  const uint32_t xl = static_cast<uint32_t>(x), xh = static_cast<uint32_t>(x >> 32);
  const uint32_t hi = __umulhi(xl, 0x133111ebu) + xl * 0x94d049bbu + xh * 0x133111ebu;  // (x * C2) >> 32
  const uint32_t hh = hi ^ (hi >> 31);
  const uint32_t th = static_cast<uint32_t>(T >> 32);
  if (hh != th) return hh > th;
  return splitmix64(h1) >= T;
}
#endif

/// detail::dropout_key (model.hpp:164-171).
__host__ __device__ __forceinline__ uint64_t dropout_key(uint64_t seed, int dp, uint64_t gstep, int layer) {
  return hash_combine(hash_combine(hash_combine(hash_combine(seed, 0xd509), static_cast<uint64_t>(dp)), gstep),
                      static_cast<uint64_t>(layer));
}

/// rng.hpp:73-76 as a double.
__host__ __device__ __forceinline__ double element_unit(uint64_t key, uint64_t i, uint64_t j) {
  const uint64_t h = splitmix64(hash_combine(hash_combine(key, i), j));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

}  // namespace ggb
