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
  const unsigned long long P01 = 184467440737095520ull;  // int(0.01 * 2**64) as Python computes it
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

namespace gw {

__device__ __forceinline__ unsigned long long wl_h2(unsigned long long a, unsigned long long b) {
  return wl_mix(wl_mix(a) ^ b);
}
__device__ __forceinline__ unsigned long long wl_h3(unsigned long long a, unsigned long long b, unsigned long long c) {
  return wl_mix(wl_h2(a, b) ^ c);
}
__device__ __forceinline__ unsigned long long wl_h4(unsigned long long a, unsigned long long b, unsigned long long c,
                                                    unsigned long long d) {
  return wl_mix(wl_h3(a, b, c) ^ d);
}

// C4 (ITS divergence), the recipe of workloads.py:c4_text.  Per iteration `it`,
// for b, for w: the lanes with bit 63 of h(hh,l,4) set issue single-lane
// accesses in order of h(hh,l,5), then the other lanes one wacc; every 4th
// iteration a warp barrier with a random mask; every 64th, block barriers.
// One warp per (it, b, w) group; its 32 (or 33) events sit at a closed-form
// offset, so the whole trace is generated in parallel.
struct C4Params {
  uint32_t B, W, L, iters;
  unsigned long long words_per_block, seed;
};

__device__ __forceinline__ uint64_t c4_iter_base(const C4Params& p, uint64_t it) {
  // events before iteration it: per iteration B*W*32 accesses, B*W warp barriers
  // when it%4==3, B block barriers when it%64==63
  const uint64_t g = (uint64_t)p.B * p.W;
  const uint64_t nbar_w = (it + 0) / 4;   // iterations j < it with j%4==3
  const uint64_t nbar_b = (it + 0) / 64;  // iterations j < it with j%64==63
  return it * g * 32ull + nbar_w * g + nbar_b * p.B;
}

__global__ void k_gen_c4(C4Params p, unsigned long long* key, uint32_t* tidop, uint32_t* instr) {
  const int lane = threadIdx.x & 31;
  const uint64_t g = (uint64_t)p.B * p.W;
  const uint64_t ngroups = g * p.iters;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // thresholds exactly as Python computes int(x * 2**64)
  const unsigned long long T99 = 18262276632972455936ull;
  const unsigned long long T9999 = 18444899399302180864ull;
  const unsigned long long T60 = 11068046444225730560ull;
  for (uint64_t gi = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < ngroups; gi += nwarps) {
    const uint64_t it = gi / g, bw = gi % g;
    const uint32_t b = (uint32_t)(bw / p.W), w = (uint32_t)(bw % p.W);
    const uint64_t base = c4_iter_base(p, it) + bw * (32ull + ((it % 4) == 3 ? 1ull : 0ull));
    const unsigned long long hh = wl_h4(p.seed, it, b, w);
    const unsigned long long words = (unsigned long long)p.B * p.words_per_block;
    const uint32_t l = (uint32_t)lane;
    // word(l)
    const unsigned long long x = wl_h3(hh, l, 1ull);
    const unsigned long long own = (unsigned long long)b * p.words_per_block +
                                   (((unsigned long long)p.L * p.W * it + (unsigned long long)p.L * w + l) % p.words_per_block);
    unsigned long long word;
    if (x < T99) word = own;
    else if (x < T9999) word = (unsigned long long)b * p.words_per_block + wl_h2(x, 2ull) % p.words_per_block;
    else word = wl_h2(x, 3ull) % words;
    const bool single = (wl_h3(hh, l, 4ull) >> 63) & 1ull;
    const unsigned long long ok = wl_h3(hh, l, 5ull);
    const bool isw = (hh >> 7) & 1ull;
    const uint32_t smask = __ballot_sync(0xffffffffu, single);
    const uint32_t nsingle = __popc(smask);
    // rank among the single lanes by (order key, lane): every lane runs the shuffles
    uint32_t r = 0;
    for (int o = 0; o < 32; o++) {
      const unsigned long long ko = __shfl_sync(0xffffffffu, ok, o);
      if (((smask >> o) & 1u) && (ko < ok || (ko == ok && o < lane))) r++;
    }
    const uint32_t pos = single ? r : nsingle + __popc(~smask & ((1u << lane) - 1u));
    const uint64_t e = base + pos;
    key[e] = 4ull * word;
    const uint32_t flat = (b * p.W + w) * p.L + l;
    if (single) {
      tidop[e] = flat | ((isw ? GW_K_WRITE : GW_K_READ) << GW_OP_SHIFT);
      instr[e] = 20u + l;
    } else {
      const bool cont = pos > nsingle;
      tidop[e] = flat | ((isw ? GW_K_READ : GW_K_WRITE) << GW_OP_SHIFT) | (cont ? GW_F_CONT : 0u);
      instr[e] = 19u;
    }
    if ((it % 4) == 3 && lane == 0) {
      uint32_t m = 0;
      for (uint32_t q = 0; q < 32; q++)
        if (wl_h3(hh, q, 6ull) < T60) m |= 1u << q;
      if (m == 0) m = 1;
      key[base + 32] = ((unsigned long long)b << 32) | w;  // as the parser encodes `bar warp b w m`
      tidop[base + 32] = ((b * p.W + w) * p.L) | (GW_K_BARRIER << GW_OP_SHIFT) | GW_F_WARPBAR;
      instr[base + 32] = m;
    }
    if ((it % 64) == 63 && bw == 0) {  // block barriers after all warps of the iteration
      const uint64_t bb = c4_iter_base(p, it) + g * (32ull + ((it % 4) == 3 ? 1ull : 0ull));
      for (uint32_t q = lane; q < p.B; q += 32) {
        key[bb + q] = 0;
        tidop[bb + q] = (q * p.W * p.L) | (GW_K_BARRIER << GW_OP_SHIFT);
        instr[bb + q] = 0;
      }
    }
  }
}

}  // namespace gw

namespace gw {

// C3 (spin-lock critical sections), the recipe of workloads.py:c3_text.  Per
// iteration `it`, for b, for w (group g = (it*B + b)*W + w): a full-mask rd
// then wr wacc on the warp's private region, a warp barrier, lane 0 polls the
// lock word with 0-3 failed-CAS atomic reads, acquires lock k = hh % locks,
// accesses 1-4 words of lock k's region, fences, releases, a warp barrier;
// 1 % of groups add an atomic counter write (lane 1), 0.1 % an unprotected
// write into lock k's region (lane 1); block barriers after every 16th
// iteration.  Group offsets come from the host (workloads.c3_group_offsets);
// one warp writes one group.
struct C3Params {
  uint32_t B, W, L, iters, locks, region, priv;
  unsigned long long seed;
};

__global__ void k_gen_c3(C3Params p, const unsigned long long* goff, unsigned long long* key, uint32_t* tidop,
                         uint32_t* instr) {
  const int lane = threadIdx.x & 31;
  const uint64_t gpi = (uint64_t)p.B * p.W;
  const uint64_t ngroups = gpi * p.iters;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned long long lock_base = 0x10000000ull, region_base = 0x20000000ull, counter = 0x30000000ull;
  for (uint64_t gi = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < ngroups; gi += nwarps) {
    const uint64_t it = gi / gpi, bw = gi % gpi;
    const uint32_t b = (uint32_t)(bw / p.W), w = (uint32_t)(bw % p.W);
    uint64_t e = goff[gi];
    const uint32_t f0 = (b * p.W + w) * p.L;
    const unsigned long long pw = ((unsigned long long)(b * p.W + w) * p.priv) * 4ull;
    for (uint32_t l = lane; l < p.L; l += 32) {
      const unsigned long long a = pw + (((unsigned long long)p.L * it + l) % p.priv) * 4ull;
      const uint32_t cont = l > 0 ? GW_F_CONT : 0u;
      key[e + l] = a;
      tidop[e + l] = (f0 + l) | (GW_K_READ << GW_OP_SHIFT) | cont;
      instr[e + l] = 1u;
      key[e + p.L + l] = a;
      tidop[e + p.L + l] = (f0 + l) | (GW_K_WRITE << GW_OP_SHIFT) | cont;
      instr[e + p.L + l] = 2u;
    }
    if (lane != 0) continue;
    e += 2ull * p.L;
    const uint32_t full = p.L >= 32 ? 0xffffffffu : ((1u << p.L) - 1u);
    auto push = [&](unsigned long long k, uint32_t to, uint32_t in) {
      key[e] = k; tidop[e] = to; instr[e] = in; e++;
    };
    const unsigned long long warpkey = ((unsigned long long)b << 32) | w;
    const uint32_t barto = f0 | (GW_K_BARRIER << GW_OP_SHIFT) | GW_F_WARPBAR;
    push(warpkey, barto, full);
    const unsigned long long hh = wl_h4(p.seed, it, b, w);
    const unsigned long long k = hh % p.locks;
    const unsigned long long lw = lock_base + 4ull * k;
    const uint32_t npoll = (uint32_t)((hh >> 20) % 4);
    for (uint32_t q = 0; q < npoll; q++)
      push(lw, f0 | (GW_K_READ << GW_OP_SHIFT) | GW_F_ATOMIC | GW_F_DEVICE, 3u);
    push(lw, f0 | (GW_K_ACQUIRE << GW_OP_SHIFT) | GW_F_DEVICE, 0u);
    const uint32_t nacc = 1u + (uint32_t)((hh >> 24) % 4);
    for (uint32_t a = 0; a < nacc; a++) {
      const unsigned long long x = region_base + 4ull * (k * p.region + wl_h2(hh, a) % p.region);
      const bool wr = (hh >> (28 + a)) & 1ull;
      push(x, f0 | ((wr ? GW_K_WRITE : GW_K_READ) << GW_OP_SHIFT), 4u + a);
    }
    push(0ull, f0 | (GW_K_FENCE << GW_OP_SHIFT) | GW_F_DEVICE, 0u);
    push(lw, f0 | (GW_K_RELEASE << GW_OP_SHIFT) | GW_F_DEVICE, 0u);
    push(warpkey, barto, full);
    const uint32_t l1 = 1u % p.L;
    if ((hh >> 40) % 100 == 0) {
      const bool dev = ((hh >> 48) % 10) != 0;
      push(counter, (f0 + l1) | (GW_K_WRITE << GW_OP_SHIFT) | GW_F_ATOMIC | (dev ? GW_F_DEVICE : 0u), 9u);
    }
    if ((hh >> 32) % 1000 == 0 && p.L > 1) {
      const unsigned long long x = region_base + 4ull * (k * p.region + (hh >> 8) % p.region);
      push(x, (f0 + 1) | (GW_K_WRITE << GW_OP_SHIFT), 10u);
    }
    if ((it % 16) == 15 && bw == gpi - 1)
      for (uint32_t q = 0; q < p.B; q++) push(0ull, (q * p.W * p.L) | (GW_K_BARRIER << GW_OP_SHIFT), 0u);
  }
}

}  // namespace gw
