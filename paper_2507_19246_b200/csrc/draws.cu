// draws.cu — sample parameters for keys (seed, level, k) on the device,
// bitwise identical to the host draws of the reference path:
//
//   RandomStream(seed, l, k).generator()
//     = numpy.random.default_rng(SeedSequence(seed, spawn_key=(l, k)))
//   draw_parameters -> rng.uniform(lo, hi)                (models.py:305-318)
//     = lo + (hi - lo) * next_double()   (numpy random_uniform, no FMA)
//
// Restated from the published algorithms: numpy's SeedSequence (O'Neill's
// seed_seq mixing: hashmix / mix over a 4-word pool, then generate_state),
// PCG64 seeding (pcg_setseq_128_srandom_r) and the XSL-RR 128/64 output,
// next_double = (next64 >> 11) * 2^-53.  The same __host__ __device__ code
// backs mlmcp_draw_uniform (device, one thread per sample) and
// mlmcp_draw_uniform_host (the CPU parity check against numpy in the tests).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

typedef unsigned __int128 u128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;

struct HashConst {
  uint32_t h;
};

__host__ __device__ inline uint32_t hashmix(uint32_t v, HashConst& hc) {
  v ^= hc.h;
  hc.h *= kMultA;
  v *= hc.h;
  v ^= v >> 16;
  return v;
}

__host__ __device__ inline uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// little-endian 32-bit words of a non-negative integer (0 -> one word)
__host__ __device__ inline int int_words(uint64_t v, uint32_t* w) {
  if (v == 0) {
    w[0] = 0;
    return 1;
  }
  int n = 0;
  while (v > 0) {
    w[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

// SeedSequence(seed, spawn_key=(level, k)).generate_state(4, uint64)
__host__ __device__ inline void seed_state(uint64_t seed, uint64_t level, uint64_t k,
                                           uint64_t (&out)[4]) {
  uint32_t ent[kPool + 4];
  int n = int_words(seed, ent);
  while (n < kPool) ent[n++] = 0;   // spawn keys present: pad the run entropy
  n += int_words(level, ent + n);
  n += int_words(k, ent + n);
  HashConst hc{kInitA};
  uint32_t pool[kPool];
  for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
  for (int s = kPool; s < n; ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mixw(pool[d], hashmix(ent[s], hc));
  uint32_t h = kInitB;
  uint32_t st[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % kPool];
    v ^= h;
    h *= kMultB;
    v *= h;
    v ^= v >> 16;
    st[i] = v;
  }
  for (int j = 0; j < 4; ++j) out[j] = (uint64_t)st[2 * j] | ((uint64_t)st[2 * j + 1] << 32);
}

struct Pcg64 {
  u128 state, inc;
  __host__ __device__ static u128 mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
  }
  __host__ __device__ void seed(uint64_t seed, uint64_t level, uint64_t k) {
    uint64_t s[4];
    seed_state(seed, level, k, s);
    const u128 initstate = ((u128)s[0] << 64) | s[1];
    const u128 initseq = ((u128)s[2] << 64) | s[3];
    state = 0;
    inc = (initseq << 1) | 1u;
    state = state * mult() + inc;
    state += initstate;
    state = state * mult() + inc;
  }
  __host__ __device__ uint64_t next64() {
    state = state * mult() + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __host__ __device__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

__host__ __device__ inline double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
__host__ __device__ inline double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}

__host__ __device__ inline void draw_row(uint64_t seed, uint64_t level, uint64_t k, int P,
                                         const double* lo, const double* range, double* out) {
  Pcg64 g;
  g.seed(seed, level, k);
  for (int j = 0; j < P; ++j) out[j] = add_rn(lo[j], mul_rn(range[j], g.next_double()));
}

__global__ void draw_uniform_kernel(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                                    const double* __restrict__ lo,
                                    const double* __restrict__ range, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  draw_row(seed, level, (uint64_t)(k_first + i), P, lo, range, out + (int64_t)i * P);
}

}  // namespace

int draw_uniform_device(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                        const double* lo, const double* range, double* out, cudaStream_t stream) {
  if (n == 0) return MLMCP_OK;
  draw_uniform_kernel<<<(n + 127) / 128, 128, 0, stream>>>(seed, level, k_first, n, P, lo, range,
                                                           out);
  MLMCP_LAUNCH_CHECK("draw_uniform_kernel");
  return MLMCP_OK;
}

void draw_uniform_cpu(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                      const double* lo, const double* range, double* out) {
  for (int i = 0; i < n; ++i)
    draw_row(seed, level, (uint64_t)(k_first + i), P, lo, range, out + (int64_t)i * P);
}

}  // namespace mlmcp
