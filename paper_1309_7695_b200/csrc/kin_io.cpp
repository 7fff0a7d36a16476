// kin_io.cpp — CSV/number/hash outputs of the sweep path (include/kin_io.h):
// the reference's io.hpp/format.hpp contract (format_double, fnv1a64,
// trajectory_csv, statistics_csv, sweep_csv).
//
// A table is a sequence of rows (one per grid point, or per point x grid point
// for sweeps).  kin_csv_write formats blocks of rows on a pool of host threads
// and writes the blocks in row order, so the file is byte-identical for any
// thread count; the content hash is folded over the blocks in the same order.
// Numbers: std::to_chars(chars_format::general), shortest round-trip — the
// form io.hpp:13-16 names (checked against oracle/kin_format.py and
// tests/golden/format_double.txt).
#include "../../include/kin_io.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ULL;
constexpr uint64_t kFnvPrime = 0x100000001b3ULL;

void set_err(kin_error* e, int code, const char* msg) {
  if (!e) return;
  e->code = code;
  std::snprintf(e->message, sizeof(e->message), "%s", msg);
}

inline void put_double(std::string& s, double v) {
  char b[32];
  const auto r = std::to_chars(b, b + sizeof b, v, std::chars_format::general);
  s.append(b, r.ptr);
}

// variance = m2/(n-1), 0 for n < 2 (ensemble.hpp:20-57)
inline double variance(double m2, uint64_t n) { return n < 2 ? 0.0 : m2 / static_cast<double>(n - 1); }

struct Table {
  const kin_csv_table& t;
  uint64_t rows() const {
    const uint64_t G = static_cast<uint64_t>(t.n_grid);
    return t.kind == KIN_CSV_SWEEP ? t.n_points * G : G;
  }
  void header(std::string& s) const {
    if (t.kind == KIN_CSV_SWEEP) {
      for (int a = 0; a < t.n_axes; ++a) {
        s += "param:";
        s += t.axis_names[a];
        s += ',';
      }
    }
    s += "time";
    for (int i = 0; i < t.n_species; ++i) {
      s += ',';
      s += t.species[i];
      if (t.kind != KIN_CSV_TRAJECTORY) {
        s += "_mean,";
        s += t.species[i];
        s += "_var";
      }
    }
    s += '\n';
  }
  void row(std::string& s, uint64_t r) const {
    const uint64_t G = static_cast<uint64_t>(t.n_grid), N = static_cast<uint64_t>(t.n_species);
    const uint64_t p = t.kind == KIN_CSV_SWEEP ? r / G : 0;
    const uint64_t g = r - p * G;
    if (t.kind == KIN_CSV_SWEEP) {
      for (int a = 0; a < t.n_axes; ++a) {
        put_double(s, t.point_values[p * t.n_axes + a]);
        s += ',';
      }
    }
    put_double(s, t.grid[g]);
    if (t.kind == KIN_CSV_TRAJECTORY) {
      const double* x = t.samples + g * N;
      for (uint64_t i = 0; i < N; ++i) {
        s += ',';
        put_double(s, x[i]);
      }
    } else {
      const double* mu = t.mean + (p * G + g) * N;
      const double* q = t.m2 + (p * G + g) * N;
      for (uint64_t i = 0; i < N; ++i) {
        s += ',';
        put_double(s, mu[i]);
        s += ',';
        put_double(s, variance(q[i], t.n_runs));
      }
    }
    s += '\n';
  }
};

const char* validate(const kin_csv_table* t) {
  if (!t) return "null table";
  if (t->kind < KIN_CSV_TRAJECTORY || t->kind > KIN_CSV_SWEEP) return "unknown table kind";
  if (t->n_species < 0 || t->n_grid < 0 || (t->n_species && !t->species) || (t->n_grid && !t->grid))
    return "species/grid missing";
  for (int i = 0; i < t->n_species; ++i)
    if (!t->species[i]) return "null species name";
  if (t->kind == KIN_CSV_TRAJECTORY && t->n_grid && t->n_species && !t->samples) return "samples missing";
  if (t->kind != KIN_CSV_TRAJECTORY && t->n_grid && t->n_species && (!t->mean || !t->m2)) return "mean/m2 missing";
  if (t->kind == KIN_CSV_SWEEP) {
    if (t->n_axes < 0 || (t->n_axes && !t->axis_names)) return "axis names missing";
    for (int a = 0; a < t->n_axes; ++a)
      if (!t->axis_names[a]) return "null axis name";
    if (t->n_points && t->n_axes && !t->point_values) return "point coordinates missing";
  }
  return nullptr;
}

int resolve_threads(int32_t threads) {
  if (threads > 0) return threads;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

}  // namespace

extern "C" {

int32_t kin_format_double(double v, char* buf, int32_t cap) {
  if (!buf || cap < 32) return -1;
  const auto r = std::to_chars(buf, buf + cap - 1, v, std::chars_format::general);
  *r.ptr = '\0';
  return static_cast<int32_t>(r.ptr - buf);
}

uint64_t kin_fnv1a64_update(uint64_t h, const void* bytes, uint64_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(bytes);
  for (uint64_t i = 0; i < n; ++i) h = (h ^ p[i]) * kFnvPrime;
  return h;
}

uint64_t kin_fnv1a64(const void* bytes, uint64_t n) { return kin_fnv1a64_update(kFnvOffset, bytes, n); }

int64_t kin_csv_render(const kin_csv_table* table, char* buf, int64_t cap, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (const char* m = validate(table)) {
    set_err(err, KIN_ERR_INPUT, m);
    return -1;
  }
  const Table T{*table};
  std::string s;
  T.header(s);
  const uint64_t R = T.rows();
  for (uint64_t r = 0; r < R; ++r) T.row(s, r);
  const int64_t n = static_cast<int64_t>(s.size());
  if (buf && cap >= n) std::memcpy(buf, s.data(), s.size());
  return n;
}

int kin_csv_write(const kin_csv_table* table, const char* path, int32_t threads, uint64_t* bytes_written,
                  uint64_t* content_fnv1a64, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (const char* m = validate(table)) {
    set_err(err, KIN_ERR_INPUT, m);
    return KIN_ERR_INPUT;
  }
  if (!path) {
    set_err(err, KIN_ERR_USAGE, "null path");
    return KIN_ERR_USAGE;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    set_err(err, KIN_ERR_INPUT, (std::string("cannot open ") + path).c_str());
    return KIN_ERR_INPUT;
  }
  const Table T{*table};
  const int nt = resolve_threads(threads);
  const uint64_t R = T.rows();
  const uint64_t block = 2048;  // rows per formatting task
  const uint64_t n_blocks = (R + block - 1) / block;
  std::string head;
  T.header(head);
  uint64_t h = kFnvOffset, total = 0;
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  if (content_fnv1a64) h = kin_fnv1a64_update(h, head.data(), head.size());
  total += head.size();
  // Pipeline: worker threads format blocks into a ring of slots while this
  // thread writes (and hashes) the completed blocks in row order.
  const size_t ring = static_cast<size_t>(nt) * 4;
  std::vector<std::string> slot(ring);
  std::vector<int> ready(ring, 0);                  // 1 = slot holds block `owner[slot]`
  std::vector<uint64_t> owner(ring, ~0ull);
  std::mutex mu;
  std::condition_variable cv_ready, cv_free;
  uint64_t written = 0;                              // blocks consumed by the writer
  std::atomic<uint64_t> next{0};
  std::atomic<bool> stop{false};
  auto work = [&]() {
    for (;;) {
      const uint64_t b = next.fetch_add(1);
      if (b >= n_blocks || stop.load()) return;
      const size_t k = static_cast<size_t>(b % ring);
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_free.wait(lk, [&] { return b < written + ring || stop.load(); });  // slot k released
        if (stop.load()) return;
      }
      std::string& sb = slot[k];
      sb.clear();
      const uint64_t r0 = b * block, r1 = std::min(R, r0 + block);
      for (uint64_t r = r0; r < r1; ++r) T.row(sb, r);
      {
        std::lock_guard<std::mutex> lk(mu);
        owner[k] = b;
        ready[k] = 1;
      }
      cv_ready.notify_all();
    }
  };
  std::vector<std::thread> pool;
  const int nw = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(nt), std::max<uint64_t>(n_blocks, 1)));
  for (int w = 0; w < nw; ++w) pool.emplace_back(work);
  for (uint64_t b = 0; b < n_blocks; ++b) {
    const size_t k = static_cast<size_t>(b % ring);
    {
      std::unique_lock<std::mutex> lk(mu);
      cv_ready.wait(lk, [&] { return ready[k] && owner[k] == b; });
    }
    if (ok) {
      ok = std::fwrite(slot[k].data(), 1, slot[k].size(), f) == slot[k].size();
      if (content_fnv1a64) h = kin_fnv1a64_update(h, slot[k].data(), slot[k].size());
      total += slot[k].size();
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      ready[k] = 0;
      ++written;
    }
    cv_free.notify_all();
    if (!ok) {
      stop.store(true);
      cv_free.notify_all();
      break;
    }
  }
  for (auto& th : pool) th.join();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    set_err(err, KIN_ERR_INPUT, (std::string("write failed: ") + path).c_str());
    return KIN_ERR_INPUT;
  }
  if (bytes_written) *bytes_written = total;
  if (content_fnv1a64) *content_fnv1a64 = h;
  return KIN_OK;
}

}  // extern "C"
