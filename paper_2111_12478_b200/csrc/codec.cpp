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
