// runtime.cu -- error strings, launch counting, cached device scratch and event profiling for libxpcs.so.
#include "common.cuh"
#include <algorithm>
#include <cstring>
#include "../../include/xpcs.h"

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace xpcs {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
static std::mutex g_mu;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}
void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }

void note_launch(int n) { g_launches.fetch_add(n); }
long long launches() { return g_launches.load(); }

// ---------------------------------------------------------------- scratch
struct Buf { void* p = nullptr; size_t n = 0; };
// keyed by (device, stream, slot): the legacy default stream (NULL) is the same handle on every device
static std::map<std::pair<std::pair<int, cudaStream_t>, int>, Buf> g_scratch;

void* scratch(cudaStream_t s, int slot, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    Buf& b = g_scratch[{{dev, s}, slot}];
    if (bytes == 0) bytes = 16;
    if (b.n >= bytes) return b.p;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        // no allocation inside a CUDA graph capture: run the same call once outside the capture first
        set_error("xpcs: scratch slot %d must grow to %zu bytes during graph capture (warm up outside the capture)", slot, bytes);
        return nullptr;
    }
    if (b.p) {
        cudaStreamSynchronize(s);      // the old buffer may still be in use by queued work on s
        cudaFree(b.p);
        b.p = nullptr;
        b.n = 0;
    }
    size_t want = bytes + bytes / 8;  // grow with slack
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&b.p, bytes);
        want = bytes;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        set_error("xpcs: device scratch allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
        return nullptr;
    }
    b.n = want;
    return b.p;
}

void release_scratch() {
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : g_scratch) {
        if (!kv.second.p) continue;
        cudaSetDevice(kv.first.first.first);
        cudaDeviceSynchronize();
        cudaFree(kv.second.p);
    }
    cudaSetDevice(cur);
    g_scratch.clear();
}

int sm_count() {   // of the current device (cached per device)
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load();
    if (n == 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev].store(n);
    }
    return n;
}

// ---------------------------------------------------------------- host tables
// device copies of small host tables (lag lists, species permutations), cached by content per device: the upload
// is synchronous and happens once per distinct table, so calls inside a CUDA graph capture (after one call outside
// it) carry no pageable host-memory copy.  At most kTables entries; evicting one synchronises the device.
constexpr size_t kTables = 32;
const void* host_table(const void* data, size_t bytes) {
    struct Entry { int dev; uint64_t h; std::vector<unsigned char> v; void* d; };
    static std::vector<Entry> tab;
    uint64_t h = 1469598103934665603ull ^ bytes;   // FNV-1a over 64-bit words (then the tail bytes)
    const unsigned char* p = (const unsigned char*)data;
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        uint64_t w;
        std::memcpy(&w, p + i, 8);
        h ^= w;
        h *= 1099511628211ull;
    }
    for (; i < bytes; ++i) { h ^= p[i]; h *= 1099511628211ull; }
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    for (size_t k = 0; k < tab.size(); ++k) {
        Entry& e = tab[k];
        if (e.dev == dev && e.h == h && e.v.size() == bytes && std::memcmp(e.v.data(), data, bytes) == 0) {
            if (k + 1 < tab.size()) std::rotate(tab.begin() + k, tab.begin() + k + 1, tab.end());   // most recent last
            return tab.back().d;
        }
    }
    if (tab.size() >= kTables) {
        cudaDeviceSynchronize();
        int d0 = 0;
        cudaGetDevice(&d0);
        cudaSetDevice(tab.front().dev);
        cudaFree(tab.front().d);
        cudaSetDevice(d0);
        tab.erase(tab.begin());
    }
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) e = cudaMemcpy(d, data, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (d) cudaFree(d);
        set_error("xpcs: table upload failed (%s); inside a CUDA graph capture, run the call once outside it first",
                  cudaGetErrorString(e));
        return nullptr;
    }
    tab.push_back({dev, h, std::vector<unsigned char>(p, p + bytes), d});
    return d;
}
const int32_t* lag_table(const int32_t* lags, int64_t n) {
    return (const int32_t*)host_table(lags, sizeof(int32_t) * (size_t)n);
}

// ---------------------------------------------------------------- profiling
static const char* kClassNames[KC_COUNT] = {"intensity_main", "stage", "amplitude_reduce", "g2", "xsvs", "rings", "fixup",
                                             "intensity_i8", "intensity_tc"};
struct ProfRec { std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev; };
static ProfRec g_prof[KC_COUNT];

// inside a CUDA graph capture the events become external event-record nodes: every replay re-records them, so
// profile_query() after a replay returns that replay's kernel times
static void prof_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else
        cudaEventRecord(e, s);
}
ProfScope::ProfScope(bool on, int cls, cudaStream_t s) : on_(on), cls_(cls), s_(s), a_(nullptr), b_(nullptr) {
    if (!on_) return;
    cudaEventCreate(&a_);
    cudaEventCreate(&b_);
    prof_record(a_, s_);
}
ProfScope::~ProfScope() {
    if (!on_) return;
    prof_record(b_, s_);
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof[cls_].ev.push_back({a_, b_});
}

int profile_reset() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : g_prof) {
        for (auto& p : r.ev) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
        r.ev.clear();
    }
    return 0;
}

int profile_query(int cls, const char** name, double* ms, long long* n) {
    if (cls < 0 || cls >= KC_COUNT) return XPCS_EINVAL;
    std::lock_guard<std::mutex> lk(g_mu);
    double tot = 0.0;
    for (auto& p : g_prof[cls].ev) {
        cudaEventSynchronize(p.second);
        float t = 0.f;
        if (cudaEventElapsedTime(&t, p.first, p.second) == cudaSuccess) tot += t;
        else cudaGetLastError();
    }
    if (name) *name = kClassNames[cls];
    if (ms) *ms = tot;
    if (n) *n = (long long)g_prof[cls].ev.size();
    return 0;
}

}  // namespace xpcs
