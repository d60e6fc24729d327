// Error plumbing of the C ABI (include/hopgnn.h).  No C++ exception or CUDA
// error crosses the boundary: everything becomes an hg_status plus a
// thread-local message the Python wrapper turns into the reference's
// exception types (errors.py:4-12).
#include <cstdarg>
#include <cstdio>

#include "hg_common.cuh"

static thread_local char g_err[512] = "";

int hg_fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  snprintf(g_err, sizeof(g_err), "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, what);
  return HG_ECUDA;
}

int hg_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

extern "C" const char* hg_last_error(void) { return g_err; }

extern "C" int hg_version(void) { return 1; }

extern "C" int hg_device_sync(void* stream) {
  HG_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

// ---------------------------------------------------------------- accounting
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace hg {
static std::atomic<long long> g_launches{0};
static bool g_prof_on = false;
static std::mutex g_prof_mu;
struct SiteEvents {
  std::vector<cudaEvent_t> beg, end;
  size_t used = 0;
  bool open = false;
};
static SiteEvents g_sites[PROF_NSITES];

void count_launch(int n) { g_launches += n; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void prof_begin(int site, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  SiteEvents& e = g_sites[site];
  if (e.used == e.beg.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    e.beg.push_back(a);
    e.end.push_back(b);
  }
  cudaEventRecord(e.beg[e.used], s);
  e.open = true;
}

void prof_end(int site, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  SiteEvents& e = g_sites[site];
  if (!e.open) return;
  cudaEventRecord(e.end[e.used], s);
  e.used++;
  e.open = false;
}
}  // namespace hg

extern "C" int hg_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(hg::g_prof_mu);
  hg::g_prof_on = on != 0;
  for (auto& e : hg::g_sites) { e.used = 0; e.open = false; }
  return HG_OK;
}

extern "C" int hg_prof_read(int site, double* total_ms, int* count) {
  if (site < 0 || site >= hg::PROF_NSITES) return hg_fail(HG_ERANGE, "bad profiling site");
  std::lock_guard<std::mutex> lk(hg::g_prof_mu);
  hg::SiteEvents& e = hg::g_sites[site];
  double t = 0;
  for (size_t i = 0; i < e.used; ++i) {
    HG_CUDA_TRY(cudaEventSynchronize(e.end[i]));
    float ms = 0;
    HG_CUDA_TRY(cudaEventElapsedTime(&ms, e.beg[i], e.end[i]));
    t += ms;
  }
  *total_ms = t;
  *count = (int)e.used;
  return HG_OK;
}

namespace hg {
__global__ void k_stamp(int64_t* slot) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = (int64_t)t;
}
}  // namespace hg

// Device timestamp (ns, %globaltimer) into *slot when the stream reaches it;
// capturable, so a graph replay's branches can be timed from inside the graph.
extern "C" int hg_stamp(int64_t* slot, void* stream) {
  hg::k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(slot);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_launch_count(long long* out, int reset) {
  *out = hg::g_launches.load();
  if (reset) hg::g_launches = 0;
  return HG_OK;
}
