// Library-level entry points: ABI version, thread-local error text, device info.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "fb_common.cuh"

namespace fb {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

// ------------------------------------------------------- launch accounting
static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_timing{false};
static std::mutex g_mu;
struct Rec {
  std::string name;
  cudaEvent_t start, stop;
};
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_free;

static cudaEvent_t take_event() {
  if (!g_free.empty()) {
    cudaEvent_t e = g_free.back();
    g_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s), slot(-1) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_timing.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r{n, take_event(), take_event()};
  cudaEventRecord(r.start, s);
  g_recs.push_back(r);
  slot = (int)g_recs.size() - 1;
}

static int debug_sync() {  // FB_DEBUG_SYNC=1: synchronise after every launch, name the failing kernel
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FB_DEBUG_SYNC");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v;
}

LaunchScope::~LaunchScope() {
  if (slot >= 0) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(g_recs[slot].stop, stream);
  }
  if (debug_sync()) {
    const cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      fprintf(stderr, "[fb] kernel %s failed: %s\n", name, cudaGetErrorString(e));
      fflush(stderr);
    }
  }
}

}  // namespace fb

extern "C" {

int64_t fb_launch_count(void) { return fb::g_launches.load(); }

void fb_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(fb::g_mu);
  for (auto& r : fb::g_recs) {
    fb::g_free.push_back(r.start);
    fb::g_free.push_back(r.stop);
  }
  fb::g_recs.clear();
  fb::g_timing.store(on != 0);
}

int fb_timing_report(char* names, int names_len, double* ms, int64_t* counts, int max_entries) {
  std::lock_guard<std::mutex> lk(fb::g_mu);
  std::map<std::string, std::pair<double, int64_t>> agg;
  for (auto& r : fb::g_recs) {
    if (cudaEventSynchronize(r.stop) != cudaSuccess) {
      fb::set_error("fb_timing_report: %s", cudaGetErrorString(cudaGetLastError()));
      return FB_ERR_CUDA;
    }
    float t = 0.f;
    cudaEventElapsedTime(&t, r.start, r.stop);
    auto& a = agg[r.name];
    a.first += t;
    a.second += 1;
  }
  int k = 0;
  std::string all;
  for (auto& kv : agg) {
    if (k >= max_entries) break;
    ms[k] = kv.second.first;
    counts[k] = kv.second.second;
    all += kv.first;
    all += '\n';
    ++k;
  }
  if (names && names_len > 0) {
    strncpy(names, all.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  return k;
}

int fb_abi_version(void) { return FB_ABI_VERSION; }

const char* fb_last_error(void) { return fb::g_last_error; }

int fb_device_info(int device, int* sm_count, int64_t* l2_bytes) {
  int sms = 0, l2 = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
  if (e != cudaSuccess) {
    fb::set_error("fb_device_info: %s", cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  if (sm_count) *sm_count = sms;
  if (l2_bytes) *l2_bytes = l2;
  return FB_OK;
}

}  // extern "C"
