// Host-side trace ingest: text -> 16-byte/event SoA, plus validate_trace.
//
// Mirrors the reference parser's accepted language, defaults and error
// messages (pkg/src/gpurace/trace.py:148-398) so that the CLI's exit codes and
// stderr text stay identical, but writes the columnar SoA of gwcp_b200.h
// directly instead of one Python object per event (~550 B/event in the
// reference).  Values the SoA cannot hold (addresses >= 2^63, more
// than 2^24 threads, instr >= 2^32, ...) are rejected with GW_E_UNSUPPORTED,
// never truncated.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>
#include <unordered_map>
#include <unordered_set>
#include <algorithm>
#include <memory>
#include <thread>

#include "../../include/gwcp_b200.h"
#include "common.h"

namespace {

typedef __int128 i128;

struct ParseError {
  int64_t line;
  std::string msg;
  int code;
};

// Python's repr() of a str token (ASCII subset; tokens never hold whitespace).
std::string py_repr(std::string_view s) {
  bool has_sq = s.find('\'') != std::string::npos;
  bool has_dq = s.find('"') != std::string::npos;
  char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == '\\') out += "\\\\";
    else if (c == (unsigned char)q) { out += '\\'; out += (char)c; }
    else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      if (c == '\t') out += "\\t";
      else if (c == '\n') out += "\\n";
      else if (c == '\r') out += "\\r";
      else { snprintf(buf, sizeof buf, "\\x%02x", c); out += buf; }
    } else out += (char)c;
  }
  out += q;
  return out;
}

std::string i128_str(i128 v) {
  if (v == 0) return "0";
  bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
  std::string s;
  while (u) { s += char('0' + (int)(u % 10)); u /= 10; }
  if (neg) s += '-';
  return std::string(s.rbegin(), s.rend());
}

// f"{v:#x}"
std::string hex_str(i128 v) {
  bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
  std::string s;
  if (u == 0) s = "0";
  while (u) { s += "0123456789abcdef"[(int)(u & 15)]; u >>= 4; }
  s += "x0";
  if (neg) s += '-';
  return std::string(s.rbegin(), s.rend());
}

int digit_val(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'z') return c - 'a' + 10;
  if (c >= 'A' && c <= 'Z') return c - 'A' + 10;
  return 99;
}

// Python int(s, base) for base in {0, 10, 16} restricted to ASCII.  Returns
// false on a syntax error (ValueError).  *overflow set if |v| >= 2^126.
bool py_int(std::string_view s, int base, i128* out, bool* overflow) {
  size_t i = 0, n = s.size();
  bool neg = false;
  *overflow = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; i++; }
  bool prefixed = false;
  if (i + 1 < n && s[i] == '0') {
    char p = s[i + 1] | 0x20;
    int pb = p == 'x' ? 16 : p == 'o' ? 8 : p == 'b' ? 2 : 0;
    if (pb && (base == 0 || base == pb)) { base = pb; i += 2; prefixed = true; }
  }
  bool base0_dec = false;
  if (base == 0) { base = 10; base0_dec = true; }
  // underscores: one allowed directly after a prefix, else only between digits
  if (prefixed && i < n && s[i] == '_') i++;
  if (i >= n) return false;
  i128 v = 0;
  bool any = false, last_us = false, nonzero_lead = false, first = true;
  for (; i < n; i++) {
    char c = s[i];
    if (c == '_') {
      if (!any || last_us) return false;
      last_us = true;
      continue;
    }
    int d = digit_val(c);
    if (d >= base) return false;
    if (first) { nonzero_lead = d != 0; first = false; }
    else if (base0_dec && !nonzero_lead && d != 0) return false;  // int("01", 0)
    any = true;
    last_us = false;
    if (v > ((i128)1 << 120)) *overflow = true;
    else v = v * base + d;
  }
  if (!any || last_us) return false;
  *out = neg ? -v : v;
  return true;
}

bool lower_starts_prefix(std::string_view t) {
  if (t.size() < 2 || t[0] != '0') return false;
  char p = t[1] | 0x20;
  return p == 'x' || p == 'b' || p == 'o';
}

// trace.py:_parse_int
i128 parse_int(std::string_view tok, int64_t line, const char* what, int base = 10) {
  i128 v;
  bool ovf;
  bool ok = lower_starts_prefix(tok) ? py_int(tok, 0, &v, &ovf) : py_int(tok, base, &v, &ovf);
  if (!ok) throw ParseError{line, std::string("bad ") + what + ": " + py_repr(tok), GW_E_PARSE};
  if (ovf) throw ParseError{line, std::string(what) + " too large for the SoA encoding", GW_E_UNSUPPORTED};
  return v;
}

inline bool is_ws(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

void split_ws(const char* b, const char* e, std::vector<std::string_view>& toks) {
  toks.clear();
  while (b < e) {
    while (b < e && is_ws((unsigned char)*b)) b++;
    const char* s = b;
    while (b < e && !is_ws((unsigned char)*b)) b++;
    if (b > s) toks.emplace_back(s, (size_t)(b - s));
  }
}

struct Cfg { int64_t blocks = 0, warps = 0, lanes = 0; };

struct Builder {
  Cfg cfg;
  bool have_cfg = false;
  std::vector<uint64_t> key;
  std::vector<uint32_t> tidop, instr;
  uint32_t group_ev_start = 0;

  uint32_t flat(int64_t b, int64_t w, int64_t l) const {
    return (uint32_t)((b * cfg.warps + w) * cfg.lanes + l);
  }
  void push(uint64_t k, uint32_t tid, uint32_t op, uint32_t ins, bool cont) {
    if (key.size() >= (1ull << 31))
      throw ParseError{0, "trace has more than 2^31 events", GW_E_UNSUPPORTED};
    key.push_back(k);
    tidop.push_back(tid | (op << GW_OP_SHIFT) | (cont ? GW_F_CONT : 0u));
    instr.push_back(ins);
  }
};

struct Tid { int64_t b, w, l; };

Tid parse_tid(std::string_view tok, const Cfg& cfg, int64_t line) {
  // tok.split(".") into exactly three parts (no vector: this runs once per event line)
  const size_t d1 = tok.find('.');
  const size_t d2 = d1 == std::string::npos ? d1 : tok.find('.', d1 + 1);
  if (d2 == std::string::npos || tok.find('.', d2 + 1) != std::string::npos)
    throw ParseError{line, "bad thread id: " + py_repr(tok), GW_E_PARSE};
  const std::string_view parts[3] = {tok.substr(0, d1), tok.substr(d1 + 1, d2 - d1 - 1), tok.substr(d2 + 1)};
  i128 b = parse_int(parts[0], line, "thread index");
  i128 w = parse_int(parts[1], line, "thread index");
  i128 l = parse_int(parts[2], line, "thread index");
  if (!(b >= 0 && b < cfg.blocks)) throw ParseError{line, "block " + i128_str(b) + " out of range", GW_E_PARSE};
  if (!(w >= 0 && w < cfg.warps)) throw ParseError{line, "warp " + i128_str(w) + " out of range", GW_E_PARSE};
  if (!(l >= 0 && l < cfg.lanes))
    throw ParseError{line, "lane " + i128_str(l) + " out of range (warp size " + std::to_string(cfg.lanes) + ")", GW_E_PARSE};
  return Tid{(int64_t)b, (int64_t)w, (int64_t)l};
}

// trace.py:_parse_loc
uint64_t parse_loc(std::string_view tok, int64_t block, int64_t line) {
  if (tok.size() < 3 || tok[1] != ':' || (tok[0] != 'g' && tok[0] != 's'))
    throw ParseError{line, "bad location: " + py_repr(tok), GW_E_PARSE};
  i128 a = parse_int(tok.substr(2), line, "address", 16);
  if (tok[0] == 'g') {
    if (a < 0 || a >= ((i128)1 << 63))
      throw ParseError{line, "global address " + hex_str(a) + " outside the SoA encoding [0, 2^63)", GW_E_UNSUPPORTED};
    return (uint64_t)a;
  }
  if (a < 0 || a >= ((i128)1 << 40))
    throw ParseError{line, "shared address " + hex_str(a) + " outside the SoA encoding [0, 2^40)", GW_E_UNSUPPORTED};
  return GW_SHARED_BIT | ((uint64_t)block << 40) | (uint64_t)a;
}

// returns 1 for device, 0 for block (trace.py:_parse_scope_word, SYSTEM -> DEVICE)
int parse_scope(std::string_view tok, int64_t line) {
  if (tok == "block") return 0;
  if (tok == "device" || tok == "system") return 1;
  throw ParseError{line, "bad scope: " + py_repr(tok), GW_E_PARSE};
}

struct Tail { bool atomic = false; int device = 0; bool has_instr = false; i128 instr = 0; };

// trace.py:_parse_access_tail
Tail parse_tail(const std::vector<std::string_view>& toks, size_t from, int64_t line) {
  Tail t;
  size_t i = from;
  while (i < toks.size()) {
    if (toks[i] == "atomic") {
      if (i + 1 >= toks.size()) throw ParseError{line, "atomic requires a scope", GW_E_PARSE};
      t.atomic = true;
      t.device = parse_scope(toks[i + 1], line);
      i += 2;
    } else if (toks[i] == "instr") {
      if (i + 1 >= toks.size()) throw ParseError{line, "instr requires a number", GW_E_PARSE};
      t.instr = parse_int(toks[i + 1], line, "instruction id");
      if (t.instr < 0) throw ParseError{line, "instruction id must be nonnegative", GW_E_PARSE};
      t.has_instr = true;
      i += 2;
    } else {
      throw ParseError{line, "unexpected token " + py_repr(toks[i]), GW_E_PARSE};
    }
  }
  return t;
}

uint32_t instr_u32(const Tail& t, int64_t line) {
  i128 v = t.has_instr ? t.instr : (i128)line;
  if (v >= ((i128)1 << 32))
    throw ParseError{line, "instruction id " + i128_str(v) + " outside the SoA encoding [0, 2^32)", GW_E_UNSUPPORTED};
  return (uint32_t)v;
}

void check_mask(i128 mask, const Cfg& cfg, int64_t line) {
  if (mask <= 0 || (cfg.lanes < 126 && mask >= ((i128)1 << cfg.lanes)))
    throw ParseError{line, "mask " + hex_str(mask) + " out of range", GW_E_PARSE};
}

void parse_line(Builder& B, std::vector<std::string_view>& toks, int64_t line) {
  Cfg& cfg = B.cfg;
  if (!B.have_cfg) {
    if (toks[0] != "config") throw ParseError{line, "first line must be a config line", GW_E_PARSE};
    std::unordered_map<std::string, i128> vals;
    for (size_t i = 1; i < toks.size(); i++) {
      size_t eq = toks[i].find('=');
      if (eq == std::string::npos) throw ParseError{line, "bad config entry " + py_repr(toks[i]), GW_E_PARSE};
      std::string k(toks[i].substr(0, eq));
      std::string_view v = toks[i].substr(eq + 1);
      vals[k] = parse_int(v, line, k.c_str());
    }
    for (const char* k : {"blocks", "warps", "lanes"})
      if (!vals.count(k)) throw ParseError{line, std::string("config missing ") + k, GW_E_PARSE};
    i128 b = vals["blocks"], w = vals["warps"], l = vals["lanes"];
    if (b < 1 || w < 1 || l < 1) throw ParseError{line, "config values must be positive", GW_E_PARSE};
    if (b * w * l > (i128)GW_TID_MASK + 1)
      throw ParseError{line, "more than 2^24 threads: outside the SoA encoding", GW_E_UNSUPPORTED};
    cfg.blocks = (int64_t)b; cfg.warps = (int64_t)w; cfg.lanes = (int64_t)l;
    B.have_cfg = true;
    return;
  }
  const std::string_view t0 = toks[0];
  if (t0 == "config") throw ParseError{line, "duplicate config line", GW_E_PARSE};
  if (t0 == "bar") {
    if (toks.size() >= 3 && toks[1] == "block") {
      i128 b = parse_int(toks[2], line, "block");
      if (!(b >= 0 && b < cfg.blocks)) throw ParseError{line, "block " + i128_str(b) + " out of range", GW_E_PARSE};
      if (toks.size() > 3) throw ParseError{line, "trailing tokens on barrier", GW_E_PARSE};
      B.push(0, B.flat((int64_t)b, 0, 0), GW_K_BARRIER, 0, false);
    } else if (toks.size() == 5 && toks[1] == "warp") {
      i128 b = parse_int(toks[2], line, "block");
      i128 w = parse_int(toks[3], line, "warp");
      i128 mask = parse_int(toks[4], line, "mask", 16);
      if (!(b >= 0 && b < cfg.blocks) || !(w >= 0 && w < cfg.warps))
        throw ParseError{line, "barrier block/warp out of range", GW_E_PARSE};
      check_mask(mask, cfg, line);
      if (cfg.lanes > 32)
        throw ParseError{line, "warp barrier with more than 32 lanes: outside the SoA encoding", GW_E_UNSUPPORTED};
      B.push(((uint64_t)b << 32) | (uint64_t)w, B.flat((int64_t)b, (int64_t)w, 0),
             GW_K_BARRIER | (GW_F_WARPBAR >> GW_OP_SHIFT), (uint32_t)mask, false);
    } else {
      throw ParseError{line, "bad barrier line", GW_E_PARSE};
    }
    return;
  }
  if (t0 == "wacc") {
    if (toks.size() < 5) throw ParseError{line, "bad wacc line", GW_E_PARSE};
    i128 b = parse_int(toks[1], line, "block");
    i128 w = parse_int(toks[2], line, "warp");
    i128 mask = parse_int(toks[3], line, "mask", 16);
    if (!(b >= 0 && b < cfg.blocks) || !(w >= 0 && w < cfg.warps))
      throw ParseError{line, "wacc block/warp out of range", GW_E_PARSE};
    check_mask(mask, cfg, line);
    uint32_t kind;
    if (toks[4] == "rd") kind = GW_K_READ;
    else if (toks[4] == "wr") kind = GW_K_WRITE;
    else throw ParseError{line, "bad access kind " + py_repr(toks[4]), GW_E_PARSE};
    std::vector<std::string_view> addrs;
    size_t i = 5;
    while (i < toks.size() && toks[i] != "atomic" && toks[i] != "instr") {
      const std::string_view a = toks[i];
      size_t s = 0;
      while (s <= a.size()) {
        size_t c = a.find(',', s);
        if (c == std::string::npos) c = a.size();
        if (c > s) addrs.push_back(a.substr(s, c - s));
        s = c + 1;
      }
      i++;
    }
    std::vector<int64_t> lanes;
    for (int64_t l = 0; l < cfg.lanes && l < 127; l++)
      if ((mask >> l) & 1) lanes.push_back(l);
    if (addrs.size() != lanes.size())
      throw ParseError{line, "wacc has " + std::to_string(addrs.size()) + " addresses for " +
                                 std::to_string(lanes.size()) + " active lanes", GW_E_PARSE};
    Tail tl = parse_tail(toks, i, line);
    uint32_t ins = instr_u32(tl, line);
    uint32_t op = kind | (tl.atomic ? (GW_F_ATOMIC >> GW_OP_SHIFT) : 0u) |
                  ((tl.atomic && tl.device) ? (GW_F_DEVICE >> GW_OP_SHIFT) : 0u);
    for (size_t k = 0; k < lanes.size(); k++) {
      uint64_t loc = parse_loc(addrs[k], (int64_t)b, line);
      B.push(loc, B.flat((int64_t)b, (int64_t)w, lanes[k]), op, ins, k > 0);
    }
    return;
  }
  Tid tid = parse_tid(t0, cfg, line);
  const std::string_view op = toks.size() > 1 ? toks[1] : std::string_view();
  uint32_t ft = B.flat(tid.b, tid.w, tid.l);
  if (op == "rd" || op == "wr") {
    if (toks.size() < 3) throw ParseError{line, "access needs a location", GW_E_PARSE};
    uint64_t loc = parse_loc(toks[2], tid.b, line);
    Tail tl = parse_tail(toks, 3, line);
    uint32_t kop = (op == "rd" ? GW_K_READ : GW_K_WRITE) |
                   (tl.atomic ? (GW_F_ATOMIC >> GW_OP_SHIFT) : 0u) |
                   ((tl.atomic && tl.device) ? (GW_F_DEVICE >> GW_OP_SHIFT) : 0u);
    B.push(loc, ft, kop, instr_u32(tl, line), false);
  } else if (op == "acq" || op == "rel") {
    if (toks.size() != 4) throw ParseError{line, "lock op needs a lock and a scope", GW_E_PARSE};
    i128 lk = parse_int(toks[2], line, "lock", 16);
    int dev = parse_scope(toks[3], line);
    if (lk < 0 || lk >= ((i128)1 << 64))
      throw ParseError{line, "lock id " + hex_str(lk) + " outside the SoA encoding [0, 2^64)", GW_E_UNSUPPORTED};
    uint32_t kop = (op == "acq" ? GW_K_ACQUIRE : GW_K_RELEASE) | (dev ? (GW_F_DEVICE >> GW_OP_SHIFT) : 0u);
    B.push((uint64_t)lk, ft, kop, 0, false);
  } else if (op == "fence") {
    if (toks.size() != 3) throw ParseError{line, "fence needs a scope", GW_E_PARSE};
    int dev = parse_scope(toks[2], line);
    B.push(0, ft, GW_K_FENCE | (dev ? (GW_F_DEVICE >> GW_OP_SHIFT) : 0u), 0, false);
  } else if (op == "end") {
    if (toks.size() != 2) throw ParseError{line, "trailing tokens on end", GW_E_PARSE};
    B.push(0, ft, GW_K_END, 0, false);
  } else {
    throw ParseError{line, "unknown event " + py_repr(op), GW_E_PARSE};
  }
}

template <class T>
T* dup_vec(const std::vector<T>& v) {
  T* p = (T*)malloc(sizeof(T) * (v.size() ? v.size() : 1));
  if (p && !v.empty()) memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}


// str.splitlines() terminators: \n \r \r\n \v \f \x1c \x1d \x1e
inline bool is_eol(unsigned char c) {
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e;
}

// Parse the lines of [p, end), numbering them from line_no + 1.  With
// stop_at_cfg, returns right after the config line (the sequential prefix of
// the parallel parse).  Returns the position reached; line_no is updated.
const char* parse_range(Builder& B, const char* p, const char* end, int64_t& line_no, bool stop_at_cfg) {
  std::vector<std::string_view> toks;
  while (p < end) {
    const char* s = p;
    while (p < end && !is_eol((unsigned char)*p)) p++;
    const char* e = p;
    if (p < end) {
      if (*p == '\r' && p + 1 < end && p[1] == '\n') p += 2;
      else p++;
    }
    line_no++;
    const char* hash = (const char*)memchr(s, '#', (size_t)(e - s));
    if (hash) e = hash;
    split_ws(s, e, toks);
    if (toks.empty()) continue;
    parse_line(B, toks, line_no);
    if (stop_at_cfg && B.have_cfg) break;
  }
  return p;
}

// lines in a chunk that ends just after a '\n' (or at the end of the text)
int64_t count_lines(const char* s, const char* e) {
  int64_t n = 0;
  for (const char* p = s; p < e; p++) {
    const unsigned char c = (unsigned char)*p;
    if (is_eol(c)) {
      n++;
      if (c == '\r' && p + 1 < e && p[1] == '\n') p++;
    }
  }
  if (e > s && !is_eol((unsigned char)e[-1])) n++;  // last line without a terminator
  return n;
}

struct Chunk {
  const char* s;
  const char* e;
  int64_t line0 = 0;
  Builder B;
  bool failed = false;
  ParseError err{0, "", 0};
  bool nomem = false;
};

int parse_threads(uint64_t len) {
  const char* env = getenv("GW_PARSE_THREADS");
  int t = env ? atoi(env) : (int)std::thread::hardware_concurrency();
  t = std::max(1, std::min(t, 64));
  const char* mc = getenv("GW_PARSE_MIN_CHUNK");  // tests: force many small chunks
  const uint64_t min_chunk = mc ? std::max<uint64_t>(1, strtoull(mc, nullptr, 10)) : (1ull << 22);  // 4 MiB
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)t, len / min_chunk));
}

template <class F>
void parallel_for(int n, F f) {
  if (n <= 0) return;
  std::vector<std::thread> th;
  for (int i = 1; i < n; i++) th.emplace_back(f, i);
  f(0);
  for (auto& t : th) t.join();
}

}  // namespace

// gw_parse_text: the sequential prefix up to the config line, then the rest in
// line-aligned chunks parsed concurrently (one Builder per chunk, line numbers
// from a parallel line count), concatenated in order.  The first error in
// text order wins, as in the sequential reference parser.
extern "C" int gw_parse_text(const char* text, uint64_t len, gw_trace* out, int64_t* err_line) {
  if (!out || (!text && len)) { gw_set_error("gw_parse_text: null argument"); return GW_E_ARG; }
  memset(out, 0, sizeof *out);
  if (err_line) *err_line = -1;
  Builder B0;
  std::vector<std::unique_ptr<Chunk>> ch;
  uint64_t total = 0;
  try {
    int64_t line_no = 0;
    const char* end = text + len;
    const char* p = parse_range(B0, text, end, line_no, true);
    if (!B0.have_cfg) throw ParseError{0, "empty trace (no config line)", GW_E_PARSE};
    const int T = parse_threads((uint64_t)(end - p));
    const uint64_t rest = (uint64_t)(end - p);
    const char* cs = p;
    for (int i = 0; i < T && cs < end; i++) {
      const char* ce = i == T - 1 ? end : p + rest * (uint64_t)(i + 1) / (uint64_t)T;
      if (ce < cs) ce = cs;
      if (ce < end) {
        const char* nl = (const char*)memchr(ce, '\n', (size_t)(end - ce));
        ce = nl ? nl + 1 : end;
      }
      auto c = std::make_unique<Chunk>();
      c->s = cs;
      c->e = ce;
      c->B.cfg = B0.cfg;
      c->B.have_cfg = true;
      ch.push_back(std::move(c));
      cs = ce;
    }
    const int nc = (int)ch.size();
    std::vector<int64_t> nlines(nc, 0);
    parallel_for(nc, [&](int i) { nlines[i] = count_lines(ch[i]->s, ch[i]->e); });
    int64_t ln = line_no;
    for (int i = 0; i < nc; i++) { ch[i]->line0 = ln; ln += nlines[i]; }
    parallel_for(nc, [&](int i) {
      Chunk& c = *ch[i];
      try {
        c.B.key.reserve((size_t)(c.e - c.s) / 8);
        c.B.tidop.reserve((size_t)(c.e - c.s) / 8);
        c.B.instr.reserve((size_t)(c.e - c.s) / 8);
        int64_t l = c.line0;
        parse_range(c.B, c.s, c.e, l, false);
      } catch (const ParseError& pe) {
        c.failed = true;
        c.err = pe;
      } catch (const std::bad_alloc&) {
        c.nomem = true;
      }
    });
    for (int i = 0; i < nc; i++) {
      if (total > (1ull << 31)) throw ParseError{0, "trace has more than 2^31 events", GW_E_UNSUPPORTED};
      if (ch[i]->nomem) throw std::bad_alloc();
      if (ch[i]->failed) throw ch[i]->err;
      total += ch[i]->B.key.size();
    }
    if (total > (1ull << 31)) throw ParseError{0, "trace has more than 2^31 events", GW_E_UNSUPPORTED};
  } catch (const ParseError& pe) {
    if (err_line) *err_line = pe.line;
    gw_set_error("line " + std::to_string(pe.line) + ": " + pe.msg);
    return pe.code;
  } catch (const std::bad_alloc&) {
    gw_set_error("gw_parse_text: out of host memory");
    return GW_E_NOMEM;
  }
  out->cfg.blocks = (uint32_t)B0.cfg.blocks;
  out->cfg.warps = (uint32_t)B0.cfg.warps;
  out->cfg.lanes = (uint32_t)B0.cfg.lanes;
  out->n_events = total;
  const size_t nz = total ? total : 1;
  out->key = (uint64_t*)malloc(sizeof(uint64_t) * nz);
  out->tidop = (uint32_t*)malloc(sizeof(uint32_t) * nz);
  out->instr = (uint32_t*)malloc(sizeof(uint32_t) * nz);
  if (!out->key || !out->tidop || !out->instr) {
    gw_trace_free(out);
    gw_set_error("gw_parse_text: out of host memory");
    return GW_E_NOMEM;
  }
  std::vector<uint64_t> off(ch.size() + 1, 0);
  for (size_t i = 0; i < ch.size(); i++) off[i + 1] = off[i] + ch[i]->B.key.size();
  parallel_for((int)ch.size(), [&](int i) {
    const Builder& b = ch[i]->B;
    const size_t k = b.key.size();
    if (!k) return;
    memcpy(out->key + off[i], b.key.data(), k * sizeof(uint64_t));
    memcpy(out->tidop + off[i], b.tidop.data(), k * sizeof(uint32_t));
    memcpy(out->instr + off[i], b.instr.data(), k * sizeof(uint32_t));
  });
  return GW_OK;
}

extern "C" void gw_trace_free(gw_trace* t) {
  if (!t) return;
  free(t->key);
  free(t->tidop);
  free(t->instr);
  t->key = nullptr; t->tidop = nullptr; t->instr = nullptr;
  t->n_events = 0;
}

extern "C" void gw_free(void* p) { free(p); }

// validate_trace (trace.py:522-601) over the SoA.  Diagnostics are returned as
// (event, code, a, b) and rendered into the reference's messages by the shim:
//   code 1 "barrier divergence: exited lane {a} in warp barrier mask"
//   code 2 "barrier divergence: no live threads in block {a}"
//   code 3 "event after end of thread {tid(a)}"
//   code 4 "shared location of block {a} used by thread {tid(b)}"
//   code 5 "reentrant acquire of lock {a:#x}"
//   code 6 "release of unheld lock {a:#x}"
//   code 7 "improperly nested release of lock {a:#x}"
extern "C" int gw_validate(const gw_trace_view* t, uint64_t* n_out, uint32_t** ev, uint32_t** code,
                           uint64_t** a, uint64_t** b) {
  if (!t || !n_out) { gw_set_error("gw_validate: null argument"); return GW_E_ARG; }
  const uint64_t W = t->cfg.warps, L = t->cfg.lanes, BS = W * L;
  const uint64_t T = (uint64_t)t->cfg.blocks * BS;
  std::vector<uint8_t> exited(T, 0);
  std::vector<uint64_t> live(t->cfg.blocks, BS);
  std::unordered_map<uint32_t, std::vector<uint64_t>> held;
  std::vector<uint32_t> oe, oc;
  std::vector<uint64_t> oa, ob;
  auto emit = [&](uint64_t i, uint32_t c, uint64_t x, uint64_t y) {
    oe.push_back((uint32_t)i); oc.push_back(c); oa.push_back(x); ob.push_back(y);
  };
  for (uint64_t i = 0; i < t->n_events; i++) {
    uint32_t to = t->tidop[i];
    uint32_t kind = (to >> GW_OP_SHIFT) & 7u;
    uint32_t tid = to & GW_TID_MASK;
    if (kind == GW_K_BARRIER) {
      if (to & GW_F_WARPBAR) {
        uint32_t mask = t->instr[i];
        for (uint64_t l = 0; l < L && l < 32; l++)
          if (((mask >> l) & 1u) && exited[tid + l]) emit(i, 1, l, 0);
      } else {
        uint64_t blk = tid / BS;
        if (live[blk] == 0) emit(i, 2, blk, 0);
      }
      continue;
    }
    if (tid >= T) { gw_set_error("gw_validate: thread index outside the configured hierarchy"); return GW_E_ARG; }
    if (exited[tid]) { emit(i, 3, tid, 0); continue; }
    bool is_access = kind <= GW_K_WRITE;
    uint64_t k = t->key[i];
    if (is_access && (k & GW_SHARED_BIT)) {
      uint64_t lb = (k >> 40) & ((1ull << 23) - 1);
      if (lb != tid / BS) emit(i, 4, lb, tid);
    }
    if (kind == GW_K_ACQUIRE) {
      auto& st = held[tid];
      bool in = false;
      for (uint64_t x : st) in |= x == k;
      if (in) emit(i, 5, k, 0);
      else st.push_back(k);
    } else if (kind == GW_K_RELEASE) {
      auto& st = held[tid];
      size_t pos = st.size();
      for (size_t j = 0; j < st.size(); j++) if (st[j] == k) { pos = j; break; }
      if (pos == st.size()) emit(i, 6, k, 0);
      else if (st.back() != k) { emit(i, 7, k, 0); st.erase(st.begin() + pos); }
      else st.pop_back();
    } else if (kind == GW_K_END) {
      exited[tid] = 1;
      live[tid / BS]--;
    }
  }
  *n_out = oe.size();
  if (ev) *ev = dup_vec(oe);
  if (code) *code = dup_vec(oc);
  if (a) *a = dup_vec(oa);
  if (b) *b = dup_vec(ob);
  return GW_OK;
}

// ---- binary SoA files (gwcp_b200.h) ----------------------------------------
namespace {
const char kSoaMagic[8] = {'G', 'W', 'S', 'O', 'A', 0, 1, 0};
struct SoaHeader {
  char magic[8];
  uint32_t blocks, warps, lanes, reserved;
  uint64_t n_events;
};
static_assert(sizeof(SoaHeader) == 32, "header layout");

bool write_all(FILE* f, const void* p, size_t n) { return n == 0 || fwrite(p, 1, n, f) == n; }
bool read_all(FILE* f, void* p, size_t n) { return n == 0 || fread(p, 1, n, f) == n; }
}  // namespace

extern "C" int gw_save_soa(const char* path, const gw_trace_view* t) {
  if (!path || !t || (t->n_events && (!t->key || !t->tidop || !t->instr))) {
    gw_set_error("gw_save_soa: null argument");
    return GW_E_ARG;
  }
  FILE* f = fopen(path, "wb");
  if (!f) { gw_set_error(std::string("gw_save_soa: cannot open ") + path); return GW_E_ARG; }
  SoaHeader h;
  memcpy(h.magic, kSoaMagic, 8);
  h.blocks = t->cfg.blocks; h.warps = t->cfg.warps; h.lanes = t->cfg.lanes; h.reserved = 0;
  h.n_events = t->n_events;
  const size_t n = (size_t)t->n_events;
  bool ok = write_all(f, &h, sizeof h) && write_all(f, t->key, n * 8) && write_all(f, t->tidop, n * 4) &&
            write_all(f, t->instr, n * 4);
  ok = (fclose(f) == 0) && ok;
  if (!ok) { gw_set_error(std::string("gw_save_soa: write failed: ") + path); return GW_E_ARG; }
  return GW_OK;
}

extern "C" int gw_load_soa(const char* path, gw_trace* out) {
  if (!path || !out) { gw_set_error("gw_load_soa: null argument"); return GW_E_ARG; }
  memset(out, 0, sizeof *out);
  FILE* f = fopen(path, "rb");
  if (!f) { gw_set_error(std::string("gw_load_soa: cannot open ") + path); return GW_E_ARG; }
  SoaHeader h;
  auto fail = [&](int code, const std::string& m) {
    fclose(f);
    gw_trace_free(out);
    gw_set_error("gw_load_soa: " + std::string(path) + ": " + m);
    return code;
  };
  if (!read_all(f, &h, sizeof h) || memcmp(h.magic, kSoaMagic, 8) != 0) return fail(GW_E_PARSE, "not a GWSOA file");
  const uint64_t T = (uint64_t)h.blocks * h.warps * h.lanes;
  if (!h.blocks || !h.warps || !h.lanes || T > (uint64_t)GW_TID_MASK + 1)
    return fail(GW_E_PARSE, "bad thread hierarchy in header");
  if (h.n_events > (1ull << 31)) return fail(GW_E_UNSUPPORTED, "more than 2^31 events");
  if (fseeko(f, 0, SEEK_END) != 0) return fail(GW_E_PARSE, "cannot seek");
  const uint64_t size = (uint64_t)ftello(f);
  if (size != sizeof h + 16ull * h.n_events) return fail(GW_E_PARSE, "file size does not match n_events");
  fseeko(f, (off_t)sizeof h, SEEK_SET);
  const size_t n = (size_t)h.n_events, nz = n ? n : 1;
  out->cfg.blocks = h.blocks; out->cfg.warps = h.warps; out->cfg.lanes = h.lanes;
  out->n_events = n;
  out->key = (uint64_t*)malloc(nz * 8);
  out->tidop = (uint32_t*)malloc(nz * 4);
  out->instr = (uint32_t*)malloc(nz * 4);
  if (!out->key || !out->tidop || !out->instr) return fail(GW_E_NOMEM, "out of host memory");
  if (!read_all(f, out->key, n * 8) || !read_all(f, out->tidop, n * 4) || !read_all(f, out->instr, n * 4))
    return fail(GW_E_PARSE, "short read");
  fclose(f);
  // the engine indexes per-thread state by these fields: keep them in range
  const uint32_t BS = h.warps * h.lanes;
  for (size_t i = 0; i < n; i++) {
    const uint32_t to = out->tidop[i];
    const uint32_t tid = to & GW_TID_MASK, kind = (to >> GW_OP_SHIFT) & 7u;
    bool bad = tid >= T || kind > GW_K_END || (to >> 31);
    if (!bad && kind == GW_K_BARRIER)
      bad = (to & GW_F_WARPBAR) ? (tid % h.lanes != 0 || h.lanes > 32) : (tid % BS != 0);
    if (bad) {
      char m[96];
      snprintf(m, sizeof m, "event %zu: tidop 0x%08x outside the encoding", i, to);
      gw_trace_free(out);
      gw_set_error("gw_load_soa: " + std::string(path) + ": " + m);
      return GW_E_PARSE;
    }
  }
  return GW_OK;
}
