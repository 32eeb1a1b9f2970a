// sbr_sceneio.cu -- native OBJ mesh reader (host code, multi-threaded).
//
// Replaces the line loop of the reference's OBJ reader (emtrace sceneio.py,
// _read_obj_arrays, sceneio.py:143-175): ASCII text, `v x y
// z` vertices, `f` polygons fan-triangulated, 1-based or negative (relative)
// indices with `v/vt/vn` tokens, `#` comments, every other keyword ignored.
// Tokens follow Python's float() / int() syntax (underscores between digits,
// inf / nan spellings, no hex) so the accepted files and the reported errors
// are the reference's.  Degenerate-triangle removal and the non-manifold
// warning stay in the Python layer (vectorised numpy over the arrays).
//
// Parallel two-pass parse: the text is cut into blocks at line boundaries;
// pass 1 counts the `v` / `f` lines and triangles of each block, a prefix sum
// gives every block its first vertex number (negative indices and range
// checks are relative to the vertices read so far), pass 2 parses the blocks
// into their slices of the output.  Each block keeps its first error; the
// earliest line's error is reported.
#include <algorithm>
#include <memory>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sbr.h"

namespace sbr {
int set_error(int code, const std::string& msg);
}  // namespace sbr

struct SbrObjMesh {
  std::vector<double> verts;  // (nv, 3)
  std::vector<int64_t> tris;  // (nt, 3), 0-based
};

namespace {

// str.split() whitespace within ASCII
inline bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\x0b' || c == '\x0c' ||
         (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }
inline char lower(char c) { return (c >= 'A' && c <= 'Z') ? (char)(c - 'A' + 'a') : c; }

// fixed-capacity token buffer (no heap traffic per number); longer tokens
// are parsed from a std::string
struct NumBuf {
  char small[64];
  std::string big;
  size_t n = 0;
  bool use_big = false;
  void push_back(char c) {
    if (!use_big && n + 1 < sizeof(small)) {
      small[n++] = c;
      return;
    }
    if (!use_big) {
      big.assign(small, n);
      use_big = true;
    }
    big.push_back(c);
  }
  const char* c_str() {
    if (use_big) return big.c_str();
    small[n] = '\0';
    return small;
  }
};

// digits with single underscores between digits (Python's numeric literals);
// appends the digits to out, returns the end or nullptr
template <typename Out>
const char* digit_run(const char* p, const char* e, Out& out) {
  if (p >= e || !is_digit(*p)) return nullptr;
  while (p < e) {
    if (is_digit(*p)) {
      out.push_back(*p++);
    } else if (*p == '_' && p + 1 < e && is_digit(p[1])) {
      ++p;
    } else {
      break;
    }
  }
  return p;
}

bool ieq(const char* p, const char* e, const char* word) {
  const size_t n = std::strlen(word);
  if ((size_t)(e - p) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (lower(p[i]) != word[i]) return false;
  return true;
}

// Python float(token) for an ASCII token without whitespace
bool py_float(const char* p, const char* e, double& out) {
  NumBuf s;
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) {
    neg = *q == '-';
    ++q;
  }
  if (ieq(q, e, "inf") || ieq(q, e, "infinity")) {
    out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(q, e, "nan")) {
    out = neg ? -NAN : NAN;
    return true;
  }
  if (neg) s.push_back('-');
  bool mant = false;
  if (q < e && is_digit(*q)) {
    q = digit_run(q, e, s);
    mant = true;
  }
  if (q < e && *q == '.') {
    s.push_back('.');
    ++q;
    if (q < e && is_digit(*q)) {
      q = digit_run(q, e, s);
      mant = true;
    }
  }
  if (!mant) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    s.push_back('e');
    ++q;
    if (q < e && (*q == '+' || *q == '-')) s.push_back(*q++);
    q = digit_run(q, e, s);
    if (!q) return false;
  }
  if (q != e) return false;
  out = std::strtod(s.c_str(), nullptr);  // correctly rounded, like float(); overflow -> inf
  return true;
}

// Python int(token) for the part before the first '/'; value saturates
// (any index beyond 2^62 is out of range anyway); `norm` = str(int(token))
bool py_int(const char* p, const char* e, int64_t& val, std::string& norm) {
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) {
    neg = *q == '-';
    ++q;
  }
  std::string digits;
  q = digit_run(q, e, digits);
  if (!q || q != e) return false;
  size_t z = 0;
  while (z + 1 < digits.size() && digits[z] == '0') ++z;
  digits = digits.substr(z);
  const bool zero = digits == "0";
  norm = (neg && !zero ? "-" : "") + digits;
  int64_t v = 0;
  for (char c : digits) {
    if (v > (INT64_C(1) << 62) / 10) {
      v = INT64_C(1) << 62;
      break;
    }
    v = v * 10 + (c - '0');
  }
  val = neg ? -v : v;
  return true;
}

struct ObjError {
  int64_t line = INT64_MAX;  // 1-based; INT64_MAX: none
  int32_t kind = 0;
  std::string detail;  // the offending token / line text
};

// error kinds (messages are formatted by the Python layer, as the reference's)
enum : int32_t {
  kVertexShort = 1,  // "vertex needs 3 coordinates"
  kVertexBad = 2,    // "bad vertex {body!r}"           (detail: stripped line body)
  kFaceShort = 3,    // "face needs at least 3 vertices"
  kFaceBadIndex = 4, // "bad face index {token!r}"      (detail: token)
  kFaceZero = 5,     // "face indices are 1-based, got 0"
  kFaceRange = 6,    // "face index {raw} out of range" (detail: str(raw))
};

struct Block {
  const char* b;
  const char* e;
  int64_t line0 = 0;        // lines before the block
  int64_t nv = 0, nt = 0;   // vertices / triangles in the block
  int64_t lines = 0;
  int64_t v0 = 0, t0 = 0;   // first vertex / triangle of the block (prefix sums)
  ObjError err;
};

// Universal newlines: "\n", "\r\n" and a lone "\r" end a line (text-mode open).
inline const char* line_end(const char* p, const char* e, const char** next) {
  const char* q = p;
  while (q < e && *q != '\n' && *q != '\r') ++q;
  if (q < e && *q == '\r' && q + 1 < e && q[1] == '\n') *next = q + 2;
  else *next = q < e ? q + 1 : e;
  return q;
}

// tokens of one line (comment stripped)
inline int split_tokens(const char* p, const char* e, const char** tb, const char** te, int cap) {
  const char* h = (const char*)std::memchr(p, '#', (size_t)(e - p));
  if (h) e = h;
  int n = 0;
  while (true) {
    while (p < e && is_ws((unsigned char)*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws((unsigned char)*p)) ++p;
    if (n < cap) {
      tb[n] = s;
      te[n] = p;
    }
    ++n;
  }
  return n;
}

constexpr int kMaxTok = 4096;  // tokens per line kept (faces with more corners are split in passes)

void count_block(Block& B) {
  const char* p = B.b;
  std::vector<const char*> tb(kMaxTok), te(kMaxTok);
  while (p < B.e) {
    const char* next;
    const char* le = line_end(p, B.e, &next);
    ++B.lines;
    const int n = split_tokens(p, le, tb.data(), te.data(), kMaxTok);
    if (n > 0 && te[0] - tb[0] == 1) {
      if (*tb[0] == 'v') ++B.nv;
      else if (*tb[0] == 'f' && n >= 4) B.nt += n - 3;
    }
    p = next;
  }
}

// all corner tokens of a face line, re-split when it has more than kMaxTok
void face_tokens(const char* p, const char* le, std::vector<const char*>& b,
                 std::vector<const char*>& e) {
  const char* h = (const char*)std::memchr(p, '#', (size_t)(le - p));
  if (h) le = h;
  b.clear();
  e.clear();
  while (true) {
    while (p < le && is_ws((unsigned char)*p)) ++p;
    if (p >= le) break;
    const char* s = p;
    while (p < le && !is_ws((unsigned char)*p)) ++p;
    b.push_back(s);
    e.push_back(p);
  }
}

void parse_block(Block& B, double* V, int64_t* T) {
  const char* p = B.b;
  int64_t line = B.line0, nv = B.v0, nt = B.t0;
  std::vector<const char*> tb(kMaxTok), te(kMaxTok), fb, fe;
  std::string norm;
  auto fail = [&](int32_t kind, std::string detail) {
    B.err.line = line;
    B.err.kind = kind;
    B.err.detail = std::move(detail);
  };
  while (p < B.e) {
    const char* next;
    const char* le = line_end(p, B.e, &next);
    ++line;
    const int n = split_tokens(p, le, tb.data(), te.data(), kMaxTok);
    if (n > 0 && te[0] - tb[0] == 1 && *tb[0] == 'v') {
      if (n < 4) return fail(kVertexShort, "");
      double x[3];
      for (int k = 0; k < 3; ++k) {
        if (!py_float(tb[k + 1], te[k + 1], x[k])) {
          // the reference reports the comment-stripped, stripped line body
          const char* h = (const char*)std::memchr(p, '#', (size_t)(le - p));
          const char* be = h ? h : le;
          const char* bb = p;
          while (bb < be && is_ws((unsigned char)*bb)) ++bb;
          while (be > bb && is_ws((unsigned char)be[-1])) --be;
          return fail(kVertexBad, std::string(bb, be));
        }
      }
      V[3 * nv] = x[0];
      V[3 * nv + 1] = x[1];
      V[3 * nv + 2] = x[2];
      ++nv;
    } else if (n > 0 && te[0] - tb[0] == 1 && *tb[0] == 'f') {
      if (n < 4) return fail(kFaceShort, "");
      const char** cb = tb.data() + 1;
      const char** ce = te.data() + 1;
      int nc = n - 1;
      if (n > kMaxTok) {
        face_tokens(p, le, fb, fe);
        cb = fb.data() + 1;
        ce = fe.data() + 1;
      }
      int64_t c0 = 0, cprev = 0;
      for (int k = 0; k < nc; ++k) {
        const char* s = cb[k];
        const char* slash = (const char*)std::memchr(s, '/', (size_t)(ce[k] - s));
        int64_t raw;
        if (!py_int(s, slash ? slash : ce[k], raw, norm)) return fail(kFaceBadIndex, std::string(s, ce[k]));
        if (raw == 0) return fail(kFaceZero, "");
        const int64_t idx = raw > 0 ? raw - 1 : nv + raw;
        if (idx < 0 || idx >= nv) return fail(kFaceRange, norm);
        if (k == 0) {
          c0 = idx;
        } else if (k >= 2) {
          T[3 * nt] = c0;
          T[3 * nt + 1] = cprev;
          T[3 * nt + 2] = idx;
          ++nt;
        }
        cprev = idx;
      }
    }
    p = next;
  }
}

}  // namespace

extern "C" {

static int obj_parse_impl(const char* text, int64_t len, SbrObjMesh** out, int64_t* err_line,
                          int32_t* err_kind, char* err_detail, int64_t detail_cap);

int sbr_obj_parse(const char* text, int64_t len, SbrObjMesh** out, int64_t* err_line,
                  int32_t* err_kind, char* err_detail, int64_t detail_cap) {
  try {
    return obj_parse_impl(text, len, out, err_line, err_kind, err_detail, detail_cap);
  } catch (const std::bad_alloc&) {
    return sbr::set_error(SBR_ERR_NOMEM, "obj: out of memory");
  } catch (...) {
    return sbr::set_error(SBR_ERR_INTERNAL, "obj: internal error");
  }
}

static int obj_parse_impl(const char* text, int64_t len, SbrObjMesh** out, int64_t* err_line,
                          int32_t* err_kind, char* err_detail, int64_t detail_cap) {
  if (!out || (!text && len > 0) || len < 0) return sbr::set_error(SBR_ERR_INVALID, "obj: bad arguments");
  *out = nullptr;
  if (err_line) *err_line = 0;
  if (err_kind) *err_kind = 0;
  const char* e = text + len;
  // blocks of >= 1 MiB cut after a line end
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 1;
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>((int64_t)hw * 4, len / (1 << 20) + 1));
  std::vector<Block> blocks;
  const char* p = text;
  for (int64_t k = 0; k < want && p < e; ++k) {
    const char* q = k + 1 == want ? e : std::min(e, text + (len * (k + 1)) / want);
    if (q < p) q = p;
    while (q < e && *q != '\n' && *q != '\r') ++q;           // to the end of that line
    if (q < e && *q == '\r' && q + 1 < e && q[1] == '\n') q += 2;
    else if (q < e) ++q;
    Block B;
    B.b = p;
    B.e = q;
    blocks.push_back(B);
    p = q;
  }
  // blocks b = t, t + nthreads, ... on host thread t; whatever a failed thread
  // creation leaves unstarted runs on the calling thread (no exception
  // crosses the C ABI)
  auto run = [&](auto fn) {
    std::vector<std::thread> th;
    const size_t nthreads = std::min<size_t>(blocks.size(), hw);
    std::atomic<bool> failed{false};  // an exception inside a worker (bad_alloc)
    auto work = [&](size_t t) {
      try {
        for (size_t b = t; b < blocks.size(); b += nthreads) fn(blocks[b]);
      } catch (...) {
        failed = true;
      }
    };
    size_t started = 0;
    try {
      for (; started < nthreads; ++started) th.emplace_back(work, started);
    } catch (...) {
    }
    for (size_t t = started; t < nthreads; ++t) work(t);
    for (auto& x : th) x.join();
    if (failed) throw std::bad_alloc();
  };
  if (blocks.size() > 1) run([](Block& B) { count_block(B); });
  else if (!blocks.empty()) count_block(blocks[0]);
  int64_t lines = 0, nv = 0, nt = 0;
  for (auto& B : blocks) {
    B.line0 = lines;
    B.v0 = nv;
    B.t0 = nt;
    lines += B.lines;
    nv += B.nv;
    nt += B.nt;
  }
  std::unique_ptr<SbrObjMesh> M(new SbrObjMesh);
  M->verts.resize(3 * (size_t)nv);  // bad_alloc -> SBR_ERR_NOMEM (sbr_obj_parse)
  M->tris.resize(3 * (size_t)nt);
  double* V = M->verts.data();
  int64_t* T = M->tris.data();
  if (blocks.size() > 1) run([&](Block& B) { parse_block(B, V, T); });
  else if (!blocks.empty()) parse_block(blocks[0], V, T);
  const ObjError* first = nullptr;
  for (auto& B : blocks)
    if (B.err.line != INT64_MAX && (!first || B.err.line < first->line)) first = &B.err;
  if (first) {
    if (err_line) *err_line = first->line;
    if (err_kind) *err_kind = first->kind;
    if (err_detail && detail_cap > 0) {
      const size_t n = std::min<size_t>(first->detail.size(), (size_t)detail_cap - 1);
      std::memcpy(err_detail, first->detail.data(), n);
      err_detail[n] = '\0';
    }
    return sbr::set_error(SBR_ERR_INVALID, "obj: parse error at line " + std::to_string(first->line));
  }
  *out = M.release();
  return SBR_OK;
}

int sbr_obj_sizes(const SbrObjMesh* m, int64_t* n_vertices, int64_t* n_triangles) {
  if (!m) return sbr::set_error(SBR_ERR_INVALID, "obj: null mesh");
  if (n_vertices) *n_vertices = (int64_t)m->verts.size() / 3;
  if (n_triangles) *n_triangles = (int64_t)m->tris.size() / 3;
  return SBR_OK;
}

int sbr_obj_copy(const SbrObjMesh* m, double* vertices, int64_t* triangles) {
  if (!m) return sbr::set_error(SBR_ERR_INVALID, "obj: null mesh");
  if (vertices && !m->verts.empty())
    std::memcpy(vertices, m->verts.data(), sizeof(double) * m->verts.size());
  if (triangles && !m->tris.empty())
    std::memcpy(triangles, m->tris.data(), sizeof(int64_t) * m->tris.size());
  return SBR_OK;
}

void sbr_obj_free(SbrObjMesh* m) { delete m; }

}  // extern "C"
