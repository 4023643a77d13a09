// Input synthesis on the device: the R-MAT edge stream of
// paper_2212_01473_b200/generate.py:rmat_edges (counter-based, so the host
// numpy generator and this kernel emit identical edges).
#include "mce_common.cuh"
#include "mce_b200.h"

namespace {

__device__ __forceinline__ uint64_t scramble(uint64_t x, int scale, uint64_t k1, uint64_t k2) {
  const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
  const int s1 = scale / 2 > 1 ? scale / 2 : 1;
  const int s2 = scale / 3 > 1 ? scale / 3 : 1;
  x = (x * k1) & mask;
  x ^= x >> s1;
  x = (x * k2) & mask;
  x ^= x >> s2;
  x = (x * k1) & mask;
  return x;
}

__global__ void k_rmat(int scale, int64_t start, int64_t count, uint64_t key, uint64_t k1,
                       uint64_t k2, int64_t* __restrict__ out) {
  const double A = 0.57, AB = 0.57 + 0.19, ABC = 0.57 + 0.19 + 0.19;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = start + i;
    uint64_t u = 0, v = 0;
    for (int level = 0; level < scale; ++level) {
      const uint64_t h = mce_mix64((uint64_t)(e * scale + level) ^ key);
      const double r = (double)(h >> 11) * (1.0 / 9007199254740992.0);
      const uint64_t bit = 1ull << (scale - 1 - level);
      if (r >= AB) u |= bit;
      if ((r >= A && r < AB) || r >= ABC) v |= bit;
    }
    out[2 * i] = (int64_t)scramble(u, scale, k1, k2);
    out[2 * i + 1] = (int64_t)scramble(v, scale, k1, k2);
  }
}

}  // namespace

extern "C" int mce_gen_rmat(int scale, int64_t start, int64_t count, uint64_t seed,
                            int64_t* edges_dev, void* stream) {
  if (scale < 1 || scale > 31 || count < 0) {
    mce_set_error("gen_rmat: bad scale/count");
    return -2;
  }
  if (count == 0) return 0;
  const uint64_t key = mce_mix64(seed * 0x100ull + 2ull);
  const uint64_t k1 = mce_mix64(seed + 11ull) | 1ull;
  const uint64_t k2 = mce_mix64(seed + 13ull) | 1ull;
  int64_t g = (count + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  k_rmat<<<(int)g, 256, 0, (cudaStream_t)stream>>>(scale, start, count, key, k1, k2, edges_dev);
  mce_count_launch();
  MCE_CHECK(cudaGetLastError());
  return 0;
}
