// ingest.cpp -- native edge-list text parser (parse_edge_list, graph.py:63-118).
//
// Multi-threaded host parser for the common ASCII grammar of the reference's
// edge-list files: lines split at \n, \r\n or \r; blank lines and lines whose
// first non-blank character is '#' skipped; exactly two tokens per line,
// each [+-]?[0-9]+ with value in [0, 2^32) ("-0" is 0, as Python's int()).
// The raw (u, v) pairs are emitted in input order (self-loops included: the
// reference keeps their vertex); dense-id remapping and deduplication run on
// the device (gs_normalize_sparse).  Anything outside this grammar -- a
// malformed line, or bytes with other meanings to Python's str.splitlines /
// str.split / int() (non-ASCII, \v \f \x1c-\x1f, '_') -- returns GS_EPARSE
// with the line number, and the host falls back to the reference-exact Python
// parser, which raises the reference's ParseError (or accepts the input).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <thread>
#include <vector>

#include "../../include/gscan.h"

namespace {

struct Chunk {
  const char* lo;
  const char* hi;
  int64_t first_line = 0;  // 1-based number of the chunk's first line
  std::vector<uint32_t> u, v;
  int64_t err_line = -1;   // first failing line of this chunk
};

inline bool special(unsigned char c) {
  return c >= 0x80 || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f) || c == '_';
}

// one token [+-]?[0-9]+ -> value < 2^32; false if malformed or out of range
inline bool parse_tok(const char*& p, const char* end, uint32_t& out) {
  bool neg = false;
  if (p < end && (*p == '+' || *p == '-')) { neg = *p == '-'; ++p; }
  const char* d0 = p;
  uint64_t x = 0;
  while (p < end && *p >= '0' && *p <= '9') {
    x = x * 10 + (uint64_t)(*p - '0');
    if (x > 0xFFFFFFFFull) return false;
    ++p;
  }
  if (p == d0) return false;
  if (neg && x != 0) return false;
  out = (uint32_t)x;
  return true;
}

void parse_chunk(Chunk& c) {
  const char* p = c.lo;
  int64_t line = c.first_line;
  while (p < c.hi) {
    const char* eol = p;
    while (eol < c.hi && *eol != '\n' && *eol != '\r') ++eol;
    const char* q = p;
    while (q < eol && (*q == ' ' || *q == '\t')) ++q;
    bool ok = true;
    if (q < eol && *q != '#') {
      uint32_t a = 0, b = 0;
      ok = parse_tok(q, eol, a);
      if (ok) {
        const char* s = q;
        while (q < eol && (*q == ' ' || *q == '\t')) ++q;
        ok = q > s && parse_tok(q, eol, b);
        while (ok && q < eol && (*q == ' ' || *q == '\t')) ++q;
        ok = ok && q == eol;
      }
      if (ok) { c.u.push_back(a); c.v.push_back(b); }
    } else if (q < eol) {  // comment: its bytes still must not be special
      for (const char* r = q; r < eol; ++r) ok &= !special((unsigned char)*r);
    }
    if (!ok) { c.err_line = line; return; }
    // line break: \r\n counts once
    if (eol < c.hi && *eol == '\r' && eol + 1 < c.hi && eol[1] == '\n') p = eol + 2;
    else p = eol + 1;
    ++line;
  }
}

}  // namespace

static int parse_edge_text(const char* buf, int64_t len, int threads, uint32_t* u_out,
                           uint32_t* v_out, int64_t cap, int64_t* count, int64_t* err_line) {
  *count = 0;
  *err_line = -1;
  if (len <= 0) return GS_OK;
  // bytes that Python treats differently anywhere in the file -> exact path
  {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(buf);
    for (int64_t i = 0; i < len; ++i)
      if (special(b[i])) {
        int64_t line = 1;
        for (int64_t j = 0; j < i; ++j)
          line += (b[j] == '\n') || (b[j] == '\r' && !(j + 1 < len && b[j + 1] == '\n'));
        *err_line = line;
        return GS_EPARSE;
      }
  }
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t min_chunk = 1 << 20;
  int nch = (int)std::min<int64_t>(threads, std::max<int64_t>(1, len / min_chunk));
  std::vector<Chunk> ch(nch);
  const char* end = buf + len;
  const char* p = buf;
  for (int i = 0; i < nch; ++i) {  // cut at line breaks (never inside \r\n)
    ch[i].lo = p;
    const char* cut = (i + 1 == nch) ? end : buf + (len * (i + 1)) / nch;
    if (cut < p) cut = p;
    while (cut < end && *cut != '\n' && *cut != '\r') ++cut;
    if (cut < end) cut += (*cut == '\r' && cut + 1 < end && cut[1] == '\n') ? 2 : 1;
    ch[i].hi = cut;
    p = cut;
  }
  // first line number of every chunk: line breaks before it
  std::vector<int64_t> breaks(nch, 0);
  {
    std::vector<std::thread> ts;
    for (int i = 0; i < nch; ++i)
      ts.emplace_back([&, i] {
        int64_t k = 0;
        for (const char* r = ch[i].lo; r < ch[i].hi; ++r)
          k += (*r == '\n') || (*r == '\r' && !(r + 1 < end && r[1] == '\n'));
        breaks[i] = k;
      });
    for (auto& t : ts) t.join();
  }
  int64_t line = 1;
  for (int i = 0; i < nch; ++i) { ch[i].first_line = line; line += breaks[i]; }
  {
    std::vector<std::thread> ts;
    for (int i = 0; i < nch; ++i) ts.emplace_back([&, i] { parse_chunk(ch[i]); });
    for (auto& t : ts) t.join();
  }
  for (int i = 0; i < nch; ++i)
    if (ch[i].err_line >= 0) { *err_line = ch[i].err_line; return GS_EPARSE; }
  int64_t total = 0;
  for (auto& c : ch) total += (int64_t)c.u.size();
  *count = total;
  if (total > cap) return GS_EINVAL;
  int64_t at = 0;
  for (auto& c : ch) {
    memcpy(u_out + at, c.u.data(), 4 * c.u.size());
    memcpy(v_out + at, c.v.data(), 4 * c.v.size());
    at += (int64_t)c.u.size();
  }
  return GS_OK;
}

// ---------------------------------------------------------------------------
// Result writer (ClusteringResult.to_text, scan.py:892-904): one line per
// vertex "orig<TAB>letter<TAB>orig(cluster) | -1", multi-threaded.  role codes
// are the public ones (1 C, 3/4 M, 5 H, 6 O); cluster ids index orig_ids.

namespace {

inline int ulen(uint64_t x) {
  int k = 1;
  while (x >= 10) { x /= 10; ++k; }
  return k;
}

inline char* put_u(char* p, uint64_t x) {
  const int k = ulen(x);
  for (int i = k - 1; i >= 0; --i) { p[i] = (char)('0' + x % 10); x /= 10; }
  return p + k;
}

inline char letter(uint8_t r) {
  switch (r) {
    case 1: return 'C';
    case 3: case 4: return 'M';
    case 5: return 'H';
    case 6: return 'O';
    default: return '?';
  }
}

}  // namespace

static int format_result(int64_t n, const uint8_t* role, const int32_t* cluster,
                         const uint32_t* orig, int threads, char* out, int64_t cap,
                         int64_t* len) {
  *len = 0;
  if (n <= 0) return GS_OK;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n / 65536));
  auto line_len = [&](int64_t v) -> int64_t {
    const int32_t c = cluster[v];
    if (c >= n) return -1;
    return ulen(orig[v]) + 3 + (c >= 0 ? ulen(orig[c]) : 2) + 1;
  };
  std::vector<int64_t> part(nt + 1, 0);
  std::vector<int> bad(nt, 0);
  {
    std::vector<std::thread> ts;
    for (int t = 0; t < nt; ++t)
      ts.emplace_back([&, t] {
        int64_t s = 0;
        for (int64_t v = n * t / nt; v < n * (t + 1) / nt; ++v) {
          const int64_t l = line_len(v);
          if (l < 0) { bad[t] = 1; return; }
          s += l;
        }
        part[t + 1] = s;
      });
    for (auto& t : ts) t.join();
  }
  for (int t = 0; t < nt; ++t)
    if (bad[t]) return GS_EINVAL;
  for (int t = 0; t < nt; ++t) part[t + 1] += part[t];
  *len = part[nt];
  if (part[nt] > cap) return GS_EINVAL;
  std::vector<std::thread> ts;
  for (int t = 0; t < nt; ++t)
    ts.emplace_back([&, t] {
      char* p = out + part[t];
      for (int64_t v = n * t / nt; v < n * (t + 1) / nt; ++v) {
        p = put_u(p, orig[v]);
        *p++ = '\t';
        *p++ = letter(role[v]);
        *p++ = '\t';
        const int32_t c = cluster[v];
        if (c >= 0) p = put_u(p, orig[c]);
        else { *p++ = '-'; *p++ = '1'; }
        *p++ = '\n';
      }
    });
  for (auto& t : ts) t.join();
  return GS_OK;
}

// ---------------------------------------------------------------------------
// Parallel host copy (pageable caller arrays -> pinned staging) for the host
// CSR load: the DMA engines only stream asynchronously from pinned memory, and
// one thread's memcpy (~10 GB/s) would starve the ~55 GB/s link.
#include <omp.h>

void gs_parallel_copy(void* dst, const void* src, size_t bytes) {
  const size_t kMin = 1 << 20;
  if (bytes < 4 * kMin) {
    memcpy(dst, src, bytes);
    return;
  }
  const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(bytes / kMin)));
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
    memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  }
}

// C-ABI: no C++ exception (thread creation, vector growth) crosses the boundary.
extern "C" int gs_parse_edge_text(const char* buf, int64_t len, int threads, uint32_t* u_out,
                                  uint32_t* v_out, int64_t cap, int64_t* count,
                                  int64_t* err_line) {
  try {
    return parse_edge_text(buf, len, threads, u_out, v_out, cap, count, err_line);
  } catch (const std::bad_alloc&) {
    return GS_ENOMEM;
  } catch (...) {
    return GS_EINTERNAL;
  }
}

extern "C" int gs_format_result(int64_t n, const uint8_t* role, const int32_t* cluster,
                                const uint32_t* orig, int threads, char* out, int64_t cap,
                                int64_t* len) {
  try {
    return format_result(n, role, cluster, orig, threads, out, cap, len);
  } catch (const std::bad_alloc&) {
    return GS_ENOMEM;
  } catch (...) {
    return GS_EINTERNAL;
  }
}
