// Device-side generator of the C2 / C5 synthetic workloads:
// the same counter-based splitmix64 recipe as
// paper_2111_12478_b200/workloads.py:c2_soa, so the 1e9-event C5 trace can be
// produced directly in HBM (16 GB) instead of on the host.  Bench/test
// infrastructure; the analysis never calls it.
#pragma once
#include "walker.cuh"

namespace gw {

__device__ __forceinline__ unsigned long long wl_mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct C2Params {
  uint32_t B, W, L, P, R;
  unsigned long long words_per_block, seed;
};

// one thread per event; per phase: R*B*W*L accesses (r, b, w, l order) then B barriers
__global__ void k_gen_c2(C2Params p, unsigned long long* key, uint32_t* tidop, uint32_t* instr, uint64_t n) {
  const uint64_t acc = (uint64_t)p.R * p.B * p.W * p.L;
  const uint64_t per = acc + p.B;
  const unsigned long long P01 = 184467440737095516ull;  // int(0.01 * 2**64)
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ph = e / per, o = e % per;
    if (o >= acc) {
      const uint32_t b = (uint32_t)(o - acc);
      key[e] = 0;
      tidop[e] = (b * p.W * p.L) | (GW_K_BARRIER << GW_OP_SHIFT);
      instr[e] = 0;
      continue;
    }
    uint64_t x = o;
    const uint32_t l = (uint32_t)(x % p.L); x /= p.L;
    const uint32_t w = (uint32_t)(x % p.W); x /= p.W;
    const uint32_t b = (uint32_t)(x % p.B); x /= p.B;
    const uint32_t r = (uint32_t)x;
    unsigned long long z = 0;
    z = wl_mix(z ^ p.seed);
    z = wl_mix(z ^ ph);
    z = wl_mix(z ^ r);
    z = wl_mix(z ^ b);
    z = wl_mix(z ^ w);
    z = wl_mix(z ^ l);
    const unsigned long long hh = z;
    const unsigned long long words = (unsigned long long)p.B * p.words_per_block;
    const unsigned long long own =
        (unsigned long long)b * p.words_per_block + ((256ull * ph + (unsigned long long)p.L * w + l) % p.words_per_block);
    const unsigned long long rnd = wl_mix(wl_mix(0 ^ hh) ^ 7ull) % words;
    const unsigned long long word = hh < P01 ? rnd : own;
    const bool wr = ((ph + r + w) & 1ull) == 0;
    key[e] = word * 4ull;
    tidop[e] = ((b * p.W + w) * p.L + l) | ((wr ? GW_K_WRITE : GW_K_READ) << GW_OP_SHIFT) | (l > 0 ? GW_F_CONT : 0u);
    instr[e] = 16u * r + w;
  }
}

}  // namespace gw
