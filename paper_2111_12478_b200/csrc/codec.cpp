// Delta-varint trace encoding (gw_trace_delta, include/gwcp_b200.h): the
// compact host / on-disk form of the SoA for end-to-end analyses, decoded on
// the device (k_delta_decode, engine.cu) while later chunks are still on the
// PCIe bus.
//
// Per column (key u64, tidop u32, instr u32): d_i = x_i - x_{i-1} (mod 2^w),
// zigzag as a signed w-bit value, LEB128 varint.  Columns are cut into
// chunks of GW_DELTA_CHUNK events; every chunk records the byte offset of its
// first varint and the column value just before it (base), so chunks decode
// independently (no cross-chunk carry).  Consecutive lanes of a record differ
// by small constants (address +4, thread +1, same instr), so C2 / C5 traces
// take ~3.3 B/event (keys 1.08, tidop 1.25, instr 1.0) instead of 16.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gwcp_b200.h"
#include "common.h"

namespace {

template <class T>
inline uint64_t zigzag(T d) {
  using S = typename std::make_signed<T>::type;
  const S s = (S)d;
  return (uint64_t)(((T)s << 1) ^ (T)(s >> (sizeof(T) * 8 - 1)));
}
inline int vput(uint8_t* p, uint64_t z) {
  int n = 0;
  do {
    uint8_t b = z & 0x7F;
    z >>= 7;
    p[n++] = (uint8_t)(b | (z ? 0x80 : 0));
  } while (z);
  return n;
}
inline int vlen(uint64_t z) {
  int n = 1;
  while (z >>= 7) n++;
  return n;
}

// one column: sizes per chunk (pass 1), then bytes (pass 2), chunk-parallel
template <class T>
bool encode_col(const T* x, uint64_t n, uint64_t nch, uint8_t** bytes, uint64_t* nbytes, uint64_t** offs,
                uint64_t** base) {
  const uint64_t CH = GW_DELTA_CHUNK;
  std::vector<uint64_t> sz(nch, 0);
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto par = [&](auto&& f) {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; w++)
      th.emplace_back([&, w] {
        for (uint64_t k = w; k < nch; k += nt) f(k);
      });
    for (auto& t : th) t.join();
  };
  par([&](uint64_t k) {
    uint64_t s = 0;
    const uint64_t lo = k * CH, hi = std::min(n, lo + CH);
    T prev = lo ? x[lo - 1] : (T)0;
    for (uint64_t i = lo; i < hi; i++) {
      s += vlen(zigzag<T>((T)(x[i] - prev)));
      prev = x[i];
    }
    sz[k] = s;
  });
  *offs = (uint64_t*)malloc(8 * (nch + 1));
  *base = (uint64_t*)malloc(8 * std::max<uint64_t>(nch, 1));
  if (!*offs || !*base) return false;
  uint64_t run = 0;
  for (uint64_t k = 0; k < nch; k++) {
    (*offs)[k] = run;
    (*base)[k] = k ? (uint64_t)x[k * CH - 1] : 0;
    run += sz[k];
  }
  (*offs)[nch] = run;
  *nbytes = run;
  *bytes = (uint8_t*)malloc(std::max<uint64_t>(run, 1) + 16);
  if (!*bytes) return false;
  uint8_t* out = *bytes;
  const uint64_t* off = *offs;
  par([&](uint64_t k) {
    uint8_t* p = out + off[k];
    const uint64_t lo = k * CH, hi = std::min(n, lo + CH);
    T prev = lo ? x[lo - 1] : (T)0;
    for (uint64_t i = lo; i < hi; i++) {
      p += vput(p, zigzag<T>((T)(x[i] - prev)));
      prev = x[i];
    }
  });
  return true;
}

}  // namespace

extern "C" void gw_delta_free(gw_trace_delta* d) {
  if (!d) return;
  for (int c = 0; c < 3; c++) {
    free((void*)d->bytes[c]);
    free((void*)d->offs[c]);
    free((void*)d->base[c]);
    d->bytes[c] = nullptr;
    d->offs[c] = nullptr;
    d->base[c] = nullptr;
  }
}

extern "C" int gw_encode_delta(const gw_trace_view* t, gw_trace_delta* out) {
  if (!t || !out) { gw_set_error("gw_encode_delta: null argument"); return GW_E_ARG; }
  if (t->n_events && (!t->key || !t->tidop || !t->instr)) {
    gw_set_error("gw_encode_delta: null trace arrays");
    return GW_E_ARG;
  }
  memset(out, 0, sizeof *out);
  const uint64_t n = t->n_events;
  out->cfg = t->cfg;
  out->n_events = n;
  out->chunk = GW_DELTA_CHUNK;
  out->n_chunks = (n + GW_DELTA_CHUNK - 1) / GW_DELTA_CHUNK;
  const uint64_t nch = out->n_chunks;
  uint8_t* b[3] = {nullptr, nullptr, nullptr};
  uint64_t* o[3] = {nullptr, nullptr, nullptr};
  uint64_t* s[3] = {nullptr, nullptr, nullptr};
  bool ok = encode_col<uint64_t>(t->key, n, nch, &b[0], &out->nbytes[0], &o[0], &s[0]) &&
            encode_col<uint32_t>(t->tidop, n, nch, &b[1], &out->nbytes[1], &o[1], &s[1]) &&
            encode_col<uint32_t>(t->instr, n, nch, &b[2], &out->nbytes[2], &o[2], &s[2]);
  for (int c = 0; c < 3; c++) {
    out->bytes[c] = b[c];
    out->offs[c] = o[c];
    out->base[c] = s[c];
  }
  if (!ok) {
    gw_delta_free(out);
    gw_set_error("gw_encode_delta: out of host memory");
    return GW_E_NOMEM;
  }
  return GW_OK;
}

// ---- bit-packed residuals (gw_trace_bp, GWSOA v4) ----------------------------
// Per column and chunk of GW_DELTA_CHUNK values: blocks of 32; the block's
// first differences d_i = x_i - x_{i-1} are predicted from d_{i-1} (mode 0),
// d_{i-32} (1) or d_{i-64} (2) -- warp-structured traces repeat every record,
// or every other one -- or not at all (3); the zigzag-coded residuals are
// packed at the cheapest width b (0..31), the wider ones stored as
// exceptions.  See include/gwcp_b200.h for the byte layout.
namespace {

inline int bits_of(uint64_t z) { return z ? 64 - __builtin_clzll(z) : 0; }

template <class T>
struct BpBlock {
  uint8_t hdr = 0, xw = 0;  // header; exception value width in bytes
  int b = 0, nexc = 0;
  uint64_t z[32];
};

// choose predictor / width of one block (k = block index in its chunk)
template <class T>
void bp_choose(const T* d, uint64_t i0, int cnt, T dprev, int k, BpBlock<T>& out) {
  int best = 1 << 30;
  for (int mode = 0; mode < 4; mode++) {
    if ((mode == 1 && k < 1) || (mode == 2 && k < 2)) continue;
    uint64_t z[32];
    int hist[65] = {0};
    for (int l = 0; l < 32; l++) {
      T r = 0;
      if (l < cnt) {
        const T pred = mode == 0 ? (l == 0 ? dprev : d[i0 + l - 1])
                                 : mode == 1 ? d[i0 + l - 32] : mode == 2 ? d[i0 + l - 64] : (T)0;
        r = (T)(d[i0 + l] - pred);
      }
      z[l] = zigzag<T>(r);
      hist[bits_of(z[l])]++;
    }
    int above = 32 - hist[0];  // values wider than b
    int wmax = 0;
    for (int q = 64; q > 0; q--)
      if (hist[q]) { wmax = q; break; }
    for (int b = 0; b < 32; b++) {
      // exceptions: their count byte + width byte, a lane byte and a value of the widest one's bytes
      const int xw = (wmax + 7) / 8;
      const int cost = 4 * b + (above ? 2 + above * (1 + xw) : 0);
      if (cost < best) {
        best = cost;
        out.b = b;
        out.nexc = above;
        out.xw = (uint8_t)(above ? xw : 0);
        out.hdr = (uint8_t)((mode << 6) | (above ? 0x20 : 0) | b);
        memcpy(out.z, z, sizeof z);
      }
      above -= hist[b + 1];
    }
  }
}

// encode one chunk (values [lo, hi)) of one column into buf; returns bytes (multiple of 4)
template <class T>
uint64_t bp_chunk(const T* d, uint64_t lo, uint64_t hi, std::vector<uint8_t>& buf) {
  const int nb = (int)((hi - lo + 31) / 32);
  std::vector<BpBlock<T>> blk(nb);
  T dprev = lo ? d[lo - 1] : (T)0;
  for (int k = 0; k < nb; k++) {
    const uint64_t i0 = lo + 32ull * k;
    const int cnt = (int)std::min<uint64_t>(32, hi - i0);
    bp_choose<T>(d, i0, cnt, dprev, k, blk[k]);
    dprev = d[i0 + cnt - 1];
  }
  buf.clear();
  for (int k = 0; k < nb; k++) buf.push_back(blk[k].hdr);
  for (int k = 0; k < nb; k++)
    if (blk[k].nexc) {
      buf.push_back((uint8_t)blk[k].nexc);
      buf.push_back(blk[k].xw);
    }
  while (buf.size() % 4) buf.push_back(0);
  for (int k = 0; k < nb; k++) {  // packed words, little-endian bit order
    const int b = blk[k].b;
    std::vector<uint32_t> w(b + 1, 0);
    const uint64_t mask = (1ull << b) - 1;
    for (int l = 0; l < 32 && b; l++) {
      const uint64_t v = blk[k].z[l] & mask;
      const int off = l * b, wi = off >> 5, sh = off & 31;
      w[wi] |= (uint32_t)(v << sh);
      if (sh + b > 32) w[wi + 1] |= (uint32_t)(v >> (32 - sh));
    }
    const size_t at = buf.size();
    buf.resize(at + 4 * (size_t)b);
    if (b) memcpy(buf.data() + at, w.data(), 4 * (size_t)b);
  }
  for (int k = 0; k < nb; k++)
    if (blk[k].nexc)
      for (int l = 0; l < 32; l++)
        if (bits_of(blk[k].z[l]) > blk[k].b) buf.push_back((uint8_t)l);
  for (int k = 0; k < nb; k++)
    if (blk[k].nexc)
      for (int l = 0; l < 32; l++)
        if (bits_of(blk[k].z[l]) > blk[k].b)
          for (int q = 0; q < blk[k].xw; q++) buf.push_back((uint8_t)(blk[k].z[l] >> (8 * q)));
  while (buf.size() % 4) buf.push_back(0);
  return buf.size();
}

template <class T>
bool bp_col(const T* x, uint64_t n, uint64_t nch, uint8_t** bytes, uint64_t* nbytes, uint64_t** offs, uint64_t** base,
            uint64_t** dbase) {
  const uint64_t CH = GW_DELTA_CHUNK;
  std::vector<T> d(n);
  for (uint64_t i = 0; i < n; i++) d[i] = (T)(x[i] - (i ? x[i - 1] : (T)0));
  std::vector<std::vector<uint8_t>> parts(nch);
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; w++)
      th.emplace_back([&, w] {
        for (uint64_t k = w; k < nch; k += nt) bp_chunk<T>(d.data(), k * CH, std::min(n, (k + 1) * CH), parts[k]);
      });
    for (auto& t : th) t.join();
  }
  *offs = (uint64_t*)malloc(8 * (nch + 1));
  *base = (uint64_t*)malloc(8 * std::max<uint64_t>(nch, 1));
  *dbase = (uint64_t*)malloc(8 * std::max<uint64_t>(nch, 1));
  if (!*offs || !*base || !*dbase) return false;
  uint64_t run = 0;
  for (uint64_t k = 0; k < nch; k++) {
    (*offs)[k] = run;
    (*base)[k] = k ? (uint64_t)x[k * CH - 1] : 0;
    (*dbase)[k] = k ? (uint64_t)d[k * CH - 1] : 0;
    run += parts[k].size();
  }
  (*offs)[nch] = run;
  *nbytes = run;
  *bytes = (uint8_t*)malloc(std::max<uint64_t>(run, 1) + 16);
  if (!*bytes) return false;
  for (uint64_t k = 0; k < nch; k++)
    if (!parts[k].empty()) memcpy(*bytes + (*offs)[k], parts[k].data(), parts[k].size());
  return true;
}

}  // namespace

extern "C" void gw_bp_free(gw_trace_bp* t) {
  if (!t) return;
  for (int c = 0; c < 3; c++) {
    free((void*)t->bytes[c]);
    free((void*)t->offs[c]);
    free((void*)t->base[c]);
    free((void*)t->dbase[c]);
    t->bytes[c] = nullptr;
    t->offs[c] = nullptr;
    t->base[c] = nullptr;
    t->dbase[c] = nullptr;
  }
}

extern "C" int gw_encode_bp(const gw_trace_view* t, gw_trace_bp* out) {
  if (!t || !out) { gw_set_error("gw_encode_bp: null argument"); return GW_E_ARG; }
  if (t->n_events && (!t->key || !t->tidop || !t->instr)) {
    gw_set_error("gw_encode_bp: null trace arrays");
    return GW_E_ARG;
  }
  memset(out, 0, sizeof *out);
  const uint64_t n = t->n_events;
  out->cfg = t->cfg;
  out->n_events = n;
  out->chunk = GW_DELTA_CHUNK;
  out->n_chunks = (n + GW_DELTA_CHUNK - 1) / GW_DELTA_CHUNK;
  const uint64_t nch = out->n_chunks;
  uint8_t* b[3] = {nullptr, nullptr, nullptr};
  uint64_t *o[3] = {nullptr, nullptr, nullptr}, *s[3] = {nullptr, nullptr, nullptr}, *ds[3] = {nullptr, nullptr, nullptr};
  uint64_t kmax = 0;
  for (uint64_t i = 0; i < n; i++) kmax = std::max<uint64_t>(kmax, t->key[i]);
  out->key_bits = kmax >> 32 ? 64 : 32;  // narrow keys: 32-bit residual arithmetic, cheaper to decode
  bool ok;
  if (out->key_bits == 32) {
    std::vector<uint32_t> k32(n);
    for (uint64_t i = 0; i < n; i++) k32[i] = (uint32_t)t->key[i];
    ok = bp_col<uint32_t>(k32.data(), n, nch, &b[0], &out->nbytes[0], &o[0], &s[0], &ds[0]);
  } else {
    ok = bp_col<uint64_t>(t->key, n, nch, &b[0], &out->nbytes[0], &o[0], &s[0], &ds[0]);
  }
  ok = ok &&
            bp_col<uint32_t>(t->tidop, n, nch, &b[1], &out->nbytes[1], &o[1], &s[1], &ds[1]) &&
            bp_col<uint32_t>(t->instr, n, nch, &b[2], &out->nbytes[2], &o[2], &s[2], &ds[2]);
  for (int c = 0; c < 3; c++) {
    out->bytes[c] = b[c];
    out->offs[c] = o[c];
    out->base[c] = s[c];
    out->dbase[c] = ds[c];
  }
  if (!ok) {
    gw_bp_free(out);
    gw_set_error("gw_encode_bp: out of host memory");
    return GW_E_NOMEM;
  }
  return GW_OK;
}
