// jq_io.cu — native CSV ingest of the reference's data-io module:
// comma-separated, '.' decimal point, one row per line, optional single header row,
// key column by zero-based index (int64, sorted non-decreasing), blank lines skipped.
// Errors name the 1-based file line (ragged row, unparsable cell, non-finite value,
// unsorted keys), as the reference's contract asks.
//
// Two calls: jq_csv_scan (row / column count) then jq_csv_parse into caller buffers.
// The file is mmapped and cut into ~4 MB newline-aligned chunks; a thread pool
// counts their rows (pass 1) and parses them with std::from_chars (exact round trip,
// pass 2).  Host outputs are written in place.  Device outputs (torch CUDA tensors)
// go through a ring of pinned staging slots: a chunk is parsed into a slot and copied
// to HBM with cudaMemcpyAsync on the context stream while the threads parse the next
// chunks, so the PCIe transfer overlaps the parse.
#include <sys/mman.h>
#include <sys/stat.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "jq_internal.cuh"

namespace jq {
namespace {

struct MappedFile {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~MappedFile() {
    if (p && n) munmap(const_cast<char*>(p), n);
    if (fd >= 0) close(fd);
  }
  int open_file(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return fail(JQ_E_INVALID, std::string(path) + ": cannot open file");
    struct stat st;
    if (fstat(fd, &st) != 0) return fail(JQ_E_INVALID, std::string(path) + ": cannot stat file");
    n = (size_t)st.st_size;
    if (n == 0) return JQ_OK;
    void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) return fail(JQ_E_INVALID, std::string(path) + ": cannot map file");
    p = static_cast<const char*>(m);
    madvise(m, n, MADV_SEQUENTIAL);
    return JQ_OK;
  }
};

inline bool blank(const char* b, const char* e) {
  for (; b < e; ++b)
    if (*b != ' ' && *b != '\t' && *b != '\r') return false;
  return true;
}

struct Chunk {
  size_t b = 0, e = 0;       // byte range [b, e), newline aligned
  int64_t rows = 0;          // non-blank lines
  int64_t lines = 0;         // all lines (for line numbers)
  int64_t row0 = 0, line0 = 0;
  int64_t first_key = 0, last_key = 0;
};

struct Layout {
  std::vector<Chunk> chunks;
  size_t body = 0;         // first byte after the header line
  int64_t header_lines = 0;
  int64_t rows = 0;
  int64_t cols = 0;        // cells per line
  int64_t first_line = 0;  // line number of the first data row (for width errors)
};

int nthreads() {
  const unsigned h = std::thread::hardware_concurrency();
  int n = (int)std::max(1u, std::min(h, 64u));
  if (const char* e = getenv("JQ_IO_THREADS")) n = std::max(1, atoi(e));
  return n;
}

template <class F>
void parallel_for(int64_t count, F&& f) {
  const int nt = (int)std::min<int64_t>(nthreads(), std::max<int64_t>(count, 1));
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (int64_t i; (i = next.fetch_add(1)) < count;) f(i);
    });
  for (auto& x : th) x.join();
}

int scan(const char* path, const MappedFile& mf, int has_header, Layout* L) {
  const char* p = mf.p;
  const size_t n = mf.n;
  size_t pos = 0;
  if (has_header && n) {
    const void* nl = memchr(p, '\n', n);
    pos = nl ? (size_t)(static_cast<const char*>(nl) - p) + 1 : n;
    L->header_lines = 1;
  }
  L->body = pos;
  // width from the first non-blank data line
  int64_t line = L->header_lines;
  size_t q = pos;
  L->cols = 0;
  while (q < n) {
    const char* nl = static_cast<const char*>(memchr(p + q, '\n', n - q));
    const size_t e = nl ? (size_t)(nl - p) : n;
    ++line;
    if (!blank(p + q, p + e)) {
      L->cols = 1 + std::count(p + q, p + e, ',');
      L->first_line = line;
      break;
    }
    q = e + 1;
  }
  // ~4 MB chunks, newline aligned
  const size_t target = size_t(4) << 20;
  for (size_t b = pos; b < n;) {
    size_t e = std::min(n, b + target);
    if (e < n) {
      const void* nl = memchr(p + e, '\n', n - e);
      e = nl ? (size_t)(static_cast<const char*>(nl) - p) + 1 : n;
    }
    Chunk c;
    c.b = b;
    c.e = e;
    L->chunks.push_back(c);
    b = e;
  }
  parallel_for((int64_t)L->chunks.size(), [&](int64_t i) {
    Chunk& c = L->chunks[i];
    for (size_t s = c.b; s < c.e;) {
      const char* nl = static_cast<const char*>(memchr(p + s, '\n', c.e - s));
      const size_t e = nl ? (size_t)(nl - p) : c.e;
      ++c.lines;
      if (!blank(p + s, p + e)) ++c.rows;
      s = e + 1;
    }
  });
  int64_t r = 0, l = L->header_lines;
  for (auto& c : L->chunks) {
    c.row0 = r;
    c.line0 = l;
    r += c.rows;
    l += c.lines;
  }
  L->rows = r;
  (void)path;
  return JQ_OK;
}

// Parse chunk c into rows [0, c.rows) of (data, keys) (row-major, ncols data columns).
// Returns "" or an error message naming the line.
std::string parse_chunk(const char* path, const char* p, Chunk& c, int64_t cols, int key_col, double* data,
                        int64_t* keys) {
  const int64_t ncols = cols - (key_col >= 0 ? 1 : 0);
  int64_t r = 0, line = c.line0;
  for (size_t s = c.b; s < c.e;) {
    const char* nl = static_cast<const char*>(memchr(p + s, '\n', c.e - s));
    const size_t e = nl ? (size_t)(nl - p) : c.e;
    ++line;
    const char* b = p + s;
    const char* end = p + e;
    s = e + 1;
    if (blank(b, end)) continue;
    if (end > b && end[-1] == '\r') --end;
    int64_t col = 0, out = 0;
    const char* cell = b;
    while (true) {
      const char* comma = static_cast<const char*>(memchr(cell, ',', (size_t)(end - cell)));
      const char* ce = comma ? comma : end;
      if (col >= cols)
        return std::string(path) + ":" + std::to_string(line) + ": ragged row (more than " + std::to_string(cols) +
               " cells, expected " + std::to_string(cols) + ")";
      const char* x = cell;
      const char* xe = ce;
      while (x < xe && (*x == ' ' || *x == '\t')) ++x;
      while (xe > x && (xe[-1] == ' ' || xe[-1] == '\t')) --xe;
      if (x < xe && *x == '+') ++x;
      if (col == key_col) {
        int64_t k = 0;
        auto res = std::from_chars(x, xe, k);
        if (res.ec != std::errc() || res.ptr != xe || x == xe)
          return std::string(path) + ":" + std::to_string(line) + ": cannot parse column " + std::to_string(col) +
                 ": '" + std::string(cell, ce) + "'";
        keys[r] = k;
      } else {
        double v = 0.0;
        auto res = std::from_chars(x, xe, v);
        if (res.ec != std::errc() || res.ptr != xe || x == xe)
          return std::string(path) + ":" + std::to_string(line) + ": cannot parse column " + std::to_string(col) +
                 ": '" + std::string(cell, ce) + "'";
        if (!std::isfinite(v)) return std::string(path) + ":" + std::to_string(line) + ": non-finite value";
        data[r * ncols + out++] = v;
      }
      ++col;
      if (!comma) break;
      cell = comma + 1;
    }
    if (col != cols)
      return std::string(path) + ":" + std::to_string(line) + ": ragged row (" + std::to_string(col) +
             " cells, expected " + std::to_string(cols) + ")";
    if (keys) {
      if (r > 0 && keys[r] < keys[r - 1])
        return std::string(path) + ":" + std::to_string(line) + ": keys are not sorted non-decreasing";
      if (r == 0) c.first_key = keys[0];
      c.last_key = keys[r];
    }
    ++r;
  }
  return "";
}

}  // namespace
}  // namespace jq

using namespace jq;

extern "C" int jq_csv_scan(const char* path, int has_header, int64_t* rows, int64_t* cols) {
  JQ_NVTX("jq_csv_scan");
  if (!path || !rows || !cols) return fail(JQ_E_INVALID, "null argument");
  MappedFile mf;
  JQ_TRY(mf.open_file(path));
  Layout L;
  JQ_TRY(scan(path, mf, has_header, &L));
  *rows = L.rows;
  *cols = L.cols;
  return JQ_OK;
}

extern "C" int jq_csv_parse(jq_ctx* ctx, const char* path, int has_header, int key_col, int64_t rows, int64_t cols,
                            double* data, int64_t* keys) {
  JQ_NVTX("jq_csv_parse");
  if (!path) return fail(JQ_E_INVALID, "null path");
  if (key_col >= 0 && key_col >= cols) return fail(JQ_E_INVALID, std::string(path) + ": key column out of range");
  if (key_col >= 0 && rows > 0 && !keys) return fail(JQ_E_INVALID, "null key output");
  if (rows > 0 && cols - (key_col >= 0 ? 1 : 0) > 0 && !data) return fail(JQ_E_INVALID, "null data output");
  MappedFile mf;
  JQ_TRY(mf.open_file(path));
  Layout L;
  JQ_TRY(scan(path, mf, has_header, &L));
  if (L.rows != rows || (rows > 0 && L.cols != cols))
    return fail(JQ_E_INVALID, std::string(path) + ": file changed between scan and parse");
  if (rows == 0) return JQ_OK;
  const int64_t ncols = cols - (key_col >= 0 ? 1 : 0);
  const bool dev = is_device_ptr(data) || is_device_ptr(keys);
  const int64_t nch = (int64_t)L.chunks.size();
  std::vector<std::string> errs(nch);
  if (!dev) {
    parallel_for(nch, [&](int64_t i) {
      Chunk& c = L.chunks[i];
      errs[i] = parse_chunk(path, mf.p, c, cols, key_col, data ? data + c.row0 * ncols : nullptr,
                            keys ? keys + c.row0 : nullptr);
    });
  } else {
    // device outputs: a ring of pinned slots; chunk i parses into slot i % S once the
    // slot's previous copy has completed, then its rows are copied on the ctx stream
    if (!ctx) return fail(JQ_E_INVALID, "null context (device outputs)");
    JQ_CUDA(cudaSetDevice(ctx->device));
    int64_t max_rows = 0;
    for (auto& c : L.chunks) max_rows = std::max(max_rows, c.rows);
    const int S = std::max(2, std::min(nthreads() + 2, 32));
    const size_t slot_bytes = size_t(max_rows) * (ncols * 8 + (keys ? 8 : 0)) + 64;
    char* pinned = nullptr;
    JQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pinned), slot_bytes * S, cudaHostAllocDefault));
    std::vector<cudaEvent_t> ev(S, nullptr);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    std::mutex mu;
    std::condition_variable cv;
    std::vector<int> done(nch, 0);      // parsed
    std::vector<int> slot_free(S, 1);   // previous copy of the slot drained (host view)
    std::atomic<int64_t> next{0};
    int64_t issued = 0;                 // chunks whose copies are queued (main thread)
    std::string cuda_err;
    auto slot_ptr = [&](int64_t i) { return pinned + size_t(i % S) * slot_bytes; };
    auto worker = [&] {
      for (int64_t i; (i = next.fetch_add(1)) < nch;) {
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return slot_free[i % S] || !cuda_err.empty(); });
          if (!cuda_err.empty()) return;
          slot_free[i % S] = 0;
        }
        Chunk& c = L.chunks[i];
        char* sp = slot_ptr(i);
        double* sd = reinterpret_cast<double*>(sp);
        int64_t* sk = keys ? reinterpret_cast<int64_t*>(sp + size_t(c.rows) * ncols * 8) : nullptr;
        errs[i] = parse_chunk(path, mf.p, c, cols, key_col, sd, sk);
        {
          std::lock_guard<std::mutex> lk(mu);
          done[i] = 1;
        }
        cv.notify_all();
      }
    };
    const int nt = (int)std::min<int64_t>(nthreads(), nch);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(worker);
    // main thread: copy chunks in order as they complete; a slot is released once its
    // copy has drained (chunk i needs the slot of chunk i - S: released before waiting)
    std::vector<int64_t> inflight;  // FIFO of chunks whose copies are queued
    size_t head = 0;
    auto release = [&](int64_t j) {
      cudaEventSynchronize(ev[j % S]);
      std::lock_guard<std::mutex> lk(mu);
      slot_free[j % S] = 1;
    };
    for (int64_t i = 0; i < nch && cuda_err.empty(); ++i) {
      while (head < inflight.size() && inflight[head] <= i - S) release(inflight[head++]);
      cv.notify_all();
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return done[i] != 0; });
      }
      Chunk& c = L.chunks[i];
      char* sp = slot_ptr(i);
      cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
      if (errs[i].empty() && c.rows > 0) {
        if (ncols > 0)
          e1 = cudaMemcpyAsync(data + c.row0 * ncols, sp, size_t(c.rows) * ncols * 8, cudaMemcpyHostToDevice,
                               ctx->stream);
        if (keys)
          e2 = cudaMemcpyAsync(keys + c.row0, sp + size_t(c.rows) * ncols * 8, size_t(c.rows) * 8,
                               cudaMemcpyHostToDevice, ctx->stream);
      }
      cudaEventRecord(ev[i % S], ctx->stream);
      inflight.push_back(i);
      issued = i + 1;
      // opportunistically release drained slots; keep at most S / 2 copies in flight
      while (head < inflight.size() &&
             (cudaEventQuery(ev[inflight[head] % S]) == cudaSuccess || inflight.size() - head > size_t(S / 2)))
        release(inflight[head++]);
      cv.notify_all();
      if (e1 != cudaSuccess || e2 != cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        cuda_err = cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
      }
    }
    while (head < inflight.size()) release(inflight[head++]);
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& f : slot_free) f = 1;
      if (cuda_err.empty() && issued < nch) cuda_err = "copy loop ended early";
    }
    cv.notify_all();
    for (auto& x : th) x.join();
    cudaStreamSynchronize(ctx->stream);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFreeHost(pinned);
    if (!cuda_err.empty()) return fail(JQ_E_CUDA, "csv H2D copy: " + cuda_err);
  }
  for (int64_t i = 0; i < nch; ++i)
    if (!errs[i].empty()) return fail(JQ_E_INVALID, errs[i]);
  if (keys) {  // sortedness across chunk boundaries
    int64_t prev = 0;
    bool have = false;
    for (auto& c : L.chunks) {
      if (c.rows == 0) continue;
      if (have && c.first_key < prev) {
        // line of the chunk's first data row
        int64_t line = c.line0;
        for (size_t s = c.b; s < c.e;) {
          const char* nl = static_cast<const char*>(memchr(mf.p + s, '\n', c.e - s));
          const size_t e = nl ? (size_t)(nl - mf.p) : c.e;
          ++line;
          if (!blank(mf.p + s, mf.p + e)) break;
          s = e + 1;
        }
        return fail(JQ_E_INVALID, std::string(path) + ":" + std::to_string(line) +
                                      ": keys are not sorted non-decreasing");
      }
      prev = c.last_key;
      have = true;
    }
  }
  return JQ_OK;
}
