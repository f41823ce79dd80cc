// trace_io.cu -- native reader of the reference's JSON-lines trace format
// (workload.py:232-313 save_trace / load_trace) straight into the skeleton CSR
// the device path consumes, so multi-million-request traces never become
// Python objects.  Host code only (compiled into libprism.so).
//
// File: one catalog header line {"catalog": {"num_segments", "chunk_tokens",
// "hot_set", "sys_prefix_tokens"}}, then one request per line {"id",
// "arrival_time", "skeleton", "suffix_tokens", "reorderable"}.  The lines are
// split over the host's cores and parsed independently; validation follows
// load_trace (workload.py:270-300): missing header, bad record, duplicate id,
// decreasing arrival_time, segment outside the catalog -- each reported with
// its 1-based line number like the reference's TraceFormatError.  Numbers are
// parsed with strtod / strtoll (correctly rounded), which reproduces Python's
// float() of json.dumps output bit for bit.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/prism.h"

namespace {

struct Rec {
  int64_t id = 0, suffix = 0, sk_begin = 0, sk_end = 0, line = 0;
  double arrival = 0.0;
  uint8_t reo = 0;
  uint8_t has = 0;  // bit per required field: id, arrival, skeleton, suffix, reorderable
};

struct Parser {
  const char *p, *e;
  std::string err;

  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) p++;
  }
  bool lit(const char *s) {
    const size_t n = strlen(s);
    if ((size_t)(e - p) >= n && !memcmp(p, s, n)) {
      p += n;
      return true;
    }
    return false;
  }
  bool str(std::string *out) {  // a JSON string (escapes kept verbatim: keys are plain)
    if (p >= e || *p != '"') return false;
    const char *b = ++p;
    while (p < e && *p != '"') p += (*p == '\\') ? 2 : 1;
    if (p >= e) return false;
    if (out) out->assign(b, p - b);
    p++;
    return true;
  }
  bool number(double *d, int64_t *i, bool *integral) {
    const char *b = p;
    if (p < e && (*p == '-' || *p == '+')) p++;
    bool frac = false;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+')) {
      frac |= (*p == '.' || *p == 'e' || *p == 'E');
      p++;
    }
    if (p == b) return false;
    std::string s(b, p - b);
    char *end = nullptr;
    if (d) *d = strtod(s.c_str(), &end);
    if (i) {
      errno = 0;
      *i = frac ? (int64_t)strtod(s.c_str(), nullptr) : strtoll(s.c_str(), nullptr, 10);
    }
    if (integral) *integral = !frac;
    return true;
  }
  bool skip_value() {
    ws();
    if (p >= e) return false;
    if (*p == '"') return str(nullptr);
    if (*p == '{' || *p == '[') {
      const char open = *p, close = open == '{' ? '}' : ']';
      p++;
      ws();
      if (p < e && *p == close) {
        p++;
        return true;
      }
      for (;;) {
        if (open == '{') {
          ws();
          if (!str(nullptr)) return false;
          ws();
          if (p >= e || *p != ':') return false;
          p++;
        }
        if (!skip_value()) return false;
        ws();
        if (p < e && *p == ',') {
          p++;
          continue;
        }
        if (p < e && *p == close) {
          p++;
          return true;
        }
        return false;
      }
    }
    if (lit("true") || lit("false") || lit("null")) return true;
    return number(nullptr, nullptr, nullptr);
  }
  // an array of integers (the skeleton)
  bool int_array(std::vector<int32_t> &out, int64_t *n) {
    ws();
    if (p >= e || *p != '[') return false;
    p++;
    ws();
    *n = 0;
    if (p < e && *p == ']') {
      p++;
      return true;
    }
    for (;;) {
      ws();
      int64_t v = 0;
      bool integral = true;
      if (!number(nullptr, &v, &integral) || !integral) return false;
      out.push_back(v < INT32_MIN ? INT32_MIN : (v > INT32_MAX ? INT32_MAX : (int32_t)v));
      (*n)++;
      ws();
      if (p < e && *p == ',') {
        p++;
        continue;
      }
      if (p < e && *p == ']') {
        p++;
        return true;
      }
      return false;
    }
  }
};

struct Catalog {
  int64_t num_segments = 0, chunk_tokens = 0, sys_prefix_tokens = 0;
  std::vector<int64_t> hot;
  bool ok = false;
};

bool parse_header(const char *b, const char *e, Catalog &c, std::string &err) {
  Parser P{b, e, {}};
  P.ws();
  if (P.p >= e || *P.p != '{') return err = "expected a JSON object", false;
  P.p++;
  for (;;) {
    P.ws();
    if (P.p < e && *P.p == '}') break;
    std::string key;
    if (!P.str(&key)) return err = "bad key", false;
    P.ws();
    if (P.p >= e || *P.p != ':') return err = "expected ':'", false;
    P.p++;
    P.ws();
    if (key == "catalog") {
      if (P.p >= e || *P.p != '{') return err = "catalog is not an object", false;
      P.p++;
      int have = 0;
      for (;;) {
        P.ws();
        if (P.p < e && *P.p == '}') {
          P.p++;
          break;
        }
        std::string k2;
        if (!P.str(&k2)) return err = "bad catalog key", false;
        P.ws();
        if (P.p >= e || *P.p != ':') return err = "expected ':'", false;
        P.p++;
        P.ws();
        if (k2 == "num_segments" || k2 == "chunk_tokens" || k2 == "sys_prefix_tokens") {
          int64_t v = 0;
          if (!P.number(nullptr, &v, nullptr)) return err = "bad catalog field " + k2, false;
          (k2 == "num_segments" ? c.num_segments : k2 == "chunk_tokens" ? c.chunk_tokens : c.sys_prefix_tokens) = v;
          have |= k2 == "num_segments" ? 1 : k2 == "chunk_tokens" ? 2 : 4;
        } else if (k2 == "hot_set") {
          std::vector<int32_t> h;
          int64_t n = 0;
          if (!P.int_array(h, &n)) return err = "bad hot_set", false;
          c.hot.assign(h.begin(), h.end());
        } else if (!P.skip_value()) {
          return err = "bad catalog value", false;
        }
        P.ws();
        if (P.p < e && *P.p == ',') P.p++;
      }
      if ((have & 3) != 3) return err = "catalog lacks num_segments / chunk_tokens", false;
      c.ok = true;
    } else if (!P.skip_value()) {
      return err = "bad value", false;
    }
    P.ws();
    if (P.p < e && *P.p == ',') P.p++;
  }
  if (!c.ok) return err = "missing catalog header", false;
  return true;
}

// one request line; skeleton entries appended to sk
bool parse_request(const char *b, const char *e, Rec &r, std::vector<int32_t> &sk, std::string &err) {
  Parser P{b, e, {}};
  P.ws();
  if (P.p >= e || *P.p != '{') return err = "expected a JSON object", false;
  P.p++;
  r.sk_begin = (int64_t)sk.size();
  for (;;) {
    P.ws();
    if (P.p < e && *P.p == '}') break;
    std::string key;
    if (!P.str(&key)) return err = "bad key", false;
    P.ws();
    if (P.p >= e || *P.p != ':') return err = "expected ':'", false;
    P.p++;
    P.ws();
    if (key == "id") {
      bool integral = true;
      if (!P.number(nullptr, &r.id, &integral) || !integral) return err = "'id' is not an integer", false;
      r.has |= 1;
    } else if (key == "arrival_time") {
      if (!P.number(&r.arrival, nullptr, nullptr)) return err = "'arrival_time' is not a number", false;
      r.has |= 2;
    } else if (key == "skeleton") {
      sk.resize((size_t)r.sk_begin);  // a repeated key: the last one wins, as in json.loads
      int64_t n = 0;
      if (!P.int_array(sk, &n)) return err = "'skeleton' is not a list of integers", false;
      r.has |= 4;
    } else if (key == "suffix_tokens") {
      if (!P.number(nullptr, &r.suffix, nullptr)) return err = "'suffix_tokens' is not a number", false;
      r.has |= 8;
    } else if (key == "reorderable") {
      if (P.lit("true")) r.reo = 1;
      else if (P.lit("false")) r.reo = 0;
      else {
        double d = 0;
        if (!P.number(&d, nullptr, nullptr)) return err = "'reorderable' is not a boolean", false;
        r.reo = d != 0.0;
      }
      r.has |= 16;
    } else if (!P.skip_value()) {
      return err = "bad value for '" + key + "'", false;
    }
    P.ws();
    if (P.p < e && *P.p == ',') P.p++;
  }
  r.sk_end = (int64_t)sk.size();
  if (r.has != 31) {
    static const char *names[] = {"id", "arrival_time", "skeleton", "suffix_tokens", "reorderable"};
    for (int b2 = 0; b2 < 5; b2++)
      if (!(r.has & (1 << b2))) return err = std::string("bad request record: '") + names[b2] + "'", false;
  }
  return true;
}

}  // namespace

struct prism_trace {
  Catalog cat;
  std::vector<int64_t> ids, off;
  std::vector<double> arr;
  std::vector<int32_t> sk, sfx;
  std::vector<uint8_t> reo;
};

extern "C" {

prism_trace *prism_trace_load_jsonl(const char *path, int32_t threads) {
  FILE *f = fopen(path, "rb");
  if (!f) {
    prism_set_last_error((std::string("cannot open ") + path).c_str());
    return nullptr;
  }
  fseek(f, 0, SEEK_END);
  const long sz = ftell(f);
  fseek(f, 0, SEEK_SET);
  std::vector<char> buf((size_t)std::max(sz, 0L));
  if (sz > 0 && fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz) {
    fclose(f);
    prism_set_last_error("short read");
    return nullptr;
  }
  fclose(f);
  const char *B = buf.data(), *E = B + buf.size();
  // line starts
  std::vector<const char *> ls;
  for (const char *q = B; q < E;) {
    ls.push_back(q);
    const char *nl = (const char *)memchr(q, '\n', (size_t)(E - q));
    q = nl ? nl + 1 : E;
  }
  if (ls.empty()) {
    prism_set_last_error("TraceFormatError: empty trace file");
    return nullptr;
  }
  auto line_end = [&](size_t i) { return i + 1 < ls.size() ? ls[i + 1] : E; };
  auto *T = new prism_trace();
  std::string err;
  if (!parse_header(ls[0], line_end(0), T->cat, err)) {
    prism_set_last_error(("TraceFormatError: line 1: " + err).c_str());
    delete T;
    return nullptr;
  }
  // request lines, split over the threads
  const size_t nl = ls.size() - 1;
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min<int>(nt, (int)std::max<size_t>(1, nl / 4096)));
  std::vector<std::vector<Rec>> recs(nt);
  std::vector<std::vector<int32_t>> sks(nt);
  std::vector<std::string> errs(nt);
  std::vector<int64_t> err_line(nt, -1);
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; w++) {
    pool.emplace_back([&, w]() {
      const size_t lo = 1 + nl * (size_t)w / nt, hi = 1 + nl * (size_t)(w + 1) / nt;
      for (size_t i = lo; i < hi; i++) {
        const char *b = ls[i], *e = line_end(i);
        const char *q = b;
        while (q < e && (*q == ' ' || *q == '\t' || *q == '\r' || *q == '\n')) q++;
        if (q == e) continue;  // blank line (load_trace skips it)
        Rec r;
        r.line = (int64_t)i + 1;
        std::string em;
        if (!parse_request(b, e, r, sks[w], em)) {
          errs[w] = em;
          err_line[w] = (int64_t)i + 1;
          return;
        }
        recs[w].push_back(r);
      }
    });
  }
  for (auto &th : pool) th.join();
  // load_trace stops at the FIRST offending line whatever the check (bad
  // record, then duplicate id, decreasing arrival, unknown segment within a
  // line): find each check's first line and report the earliest
  int64_t bad_line = INT64_MAX;
  int best_rank = 99;
  std::string bad_msg;
  auto offend = [&](int64_t line, int rank, const std::string &m) {
    if (line < bad_line || (line == bad_line && rank < best_rank)) {
      bad_line = line;
      best_rank = rank;
      bad_msg = m;
    }
  };
  for (int w = 0; w < nt; w++)
    if (err_line[w] >= 0) offend(err_line[w], 0, errs[w]);
  size_t n = 0, nsk = 0;
  for (int w = 0; w < nt; w++) {
    n += recs[w].size();
    nsk += sks[w].size();
  }
  std::vector<const Rec *> all(n);
  std::vector<int> owner(n);
  {
    size_t j = 0;
    for (int w = 0; w < nt; w++)
      for (const Rec &r : recs[w]) {
        owner[j] = w;
        all[j++] = &r;
      }
  }
  {  // duplicate ids: the second occurrence of any id
    std::vector<std::pair<int64_t, int64_t>> byid(n);
    for (size_t j = 0; j < n; j++) byid[j] = {all[j]->id, (int64_t)j};
    std::sort(byid.begin(), byid.end());
    for (size_t j = 1; j < n; j++)
      if (byid[j].first == byid[j - 1].first && (j < 2 || byid[j - 2].first != byid[j].first))
        offend(all[(size_t)byid[j].second]->line, 1, "duplicate request id " + std::to_string(byid[j].first));
  }
  const int64_t S = T->cat.num_segments;
  double last = -HUGE_VAL;
  for (size_t j = 0; j < n && all[j]->line < bad_line; j++) {
    const Rec &r = *all[j];
    if (r.arrival < last) offend(r.line, 2, "arrival_time decreases");
    last = r.arrival;
    for (int64_t e = r.sk_begin; e < r.sk_end; e++) {
      const int32_t sg = sks[owner[j]][(size_t)e];
      if (sg < 0 || sg >= S) {
        offend(r.line, 3, "skeleton references unknown segment");
        break;
      }
    }
  }
  if (bad_line != INT64_MAX) {
    prism_set_last_error(("TraceFormatError: line " + std::to_string(bad_line) + ": " + bad_msg).c_str());
    delete T;
    return nullptr;
  }
  T->ids.resize(n);
  T->arr.resize(n);
  T->off.resize(n + 1);
  T->sfx.resize(n);
  T->reo.resize(n);
  T->sk.resize(nsk);
  size_t o = 0;
  for (size_t j = 0; j < n; j++) {
    const Rec &r = *all[j];
    T->ids[j] = r.id;
    T->arr[j] = r.arrival;
    T->sfx[j] = (int32_t)r.suffix;
    T->reo[j] = r.reo;
    T->off[j] = (int64_t)o;
    for (int64_t e = r.sk_begin; e < r.sk_end; e++) T->sk[o++] = sks[owner[j]][(size_t)e];
  }
  T->off[n] = (int64_t)o;
  return T;
}

// out[0] requests, [1] skeleton entries, [2] num_segments, [3] chunk_tokens,
// [4] sys_prefix_tokens, [5] hot-set size
int prism_trace_info(prism_trace *T, int64_t *out) {
  out[0] = (int64_t)T->ids.size();
  out[1] = (int64_t)T->sk.size();
  out[2] = T->cat.num_segments;
  out[3] = T->cat.chunk_tokens;
  out[4] = T->cat.sys_prefix_tokens;
  out[5] = (int64_t)T->cat.hot.size();
  return PRISM_OK;
}

int prism_trace_copy(prism_trace *T, int64_t *ids, double *arrival, int64_t *sk_off, int32_t *sk,
                     uint8_t *reorderable, int32_t *suffix, int64_t *hot_set) {
  const size_t n = T->ids.size();
  if (ids) memcpy(ids, T->ids.data(), 8 * n);
  if (arrival) memcpy(arrival, T->arr.data(), 8 * n);
  if (sk_off) memcpy(sk_off, T->off.data(), 8 * (n + 1));
  if (sk && !T->sk.empty()) memcpy(sk, T->sk.data(), 4 * T->sk.size());
  if (reorderable) memcpy(reorderable, T->reo.data(), n);
  if (suffix) memcpy(suffix, T->sfx.data(), 4 * n);
  if (hot_set && !T->cat.hot.empty()) memcpy(hot_set, T->cat.hot.data(), 8 * T->cat.hot.size());
  return PRISM_OK;
}

void prism_trace_free(prism_trace *T) { delete T; }

}  // extern "C"
