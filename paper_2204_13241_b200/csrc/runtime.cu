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
// Buffers keyed by (device, workspace, stream, slot).  A buffer that was handed out during a CUDA graph capture is
// referenced by that graph's nodes: when the slot later has to grow it is RETIRED (kept until xpcs_release) rather
// than freed, so replaying the old graph never touches freed memory.
struct Buf { void* p = nullptr; size_t n = 0; bool captured = false; };
struct ScratchKey {
    int dev, ws;
    cudaStream_t s;
    int slot;
    bool operator<(const ScratchKey& o) const {
        if (dev != o.dev) return dev < o.dev;
        if (ws != o.ws) return ws < o.ws;
        if (s != o.s) return s < o.s;
        return slot < o.slot;
    }
};
static std::map<ScratchKey, Buf> g_scratch;
static std::vector<std::pair<int, void*>> g_retired;   // (device, buffer) of grown slots that a graph may reference
static thread_local int g_ws = 0;

void set_workspace(int ws) { g_ws = ws; }

void* scratch(cudaStream_t s, int slot, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    Buf& b = g_scratch[ScratchKey{dev, g_ws, s, slot}];
    if (bytes == 0) bytes = 16;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
    if (b.n >= bytes) {
        if (capturing) b.captured = true;
        return b.p;
    }
    if (capturing) {
        // no allocation inside a CUDA graph capture: run the same call once outside the capture first
        set_error("xpcs: scratch slot %d must grow to %zu bytes during graph capture (warm up outside the capture)", slot, bytes);
        return nullptr;
    }
    if (b.p) {
        cudaStreamSynchronize(s);      // the old buffer may still be in use by queued work on s
        if (b.captured) g_retired.push_back({dev, b.p});   // a captured graph may still replay with it
        else cudaFree(b.p);
        b.p = nullptr;
        b.n = 0;
        b.captured = false;
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
        cudaSetDevice(kv.first.dev);
        cudaDeviceSynchronize();
        cudaFree(kv.second.p);
    }
    for (auto& r : g_retired) {
        cudaSetDevice(r.first);
        cudaDeviceSynchronize();
        cudaFree(r.second);
    }
    cudaSetDevice(cur);
    g_scratch.clear();
    g_retired.clear();
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
// it) carry no pageable host-memory copy.  At most kTables entries (more while every entry is pinned); an entry
// handed out during a capture on `s` is pinned (the graph holds its pointer) and never evicted before release;
// evicting an unpinned one synchronises its own device first.
constexpr size_t kTables = 32;
const void* host_table(const void* data, size_t bytes, cudaStream_t s) {
    // pinned: handed out during a graph capture (the graph holds the pointer) -> never evicted before release
    struct Entry { int dev; uint64_t h; std::vector<unsigned char> v; void* d; bool pinned; };
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
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const bool pin = cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
    for (size_t k = 0; k < tab.size(); ++k) {
        Entry& e = tab[k];
        if (e.dev == dev && e.h == h && e.v.size() == bytes && std::memcmp(e.v.data(), data, bytes) == 0) {
            if (pin) e.pinned = true;
            if (k + 1 < tab.size()) std::rotate(tab.begin() + k, tab.begin() + k + 1, tab.end());   // most recent last
            return tab.back().d;
        }
    }
    if (tab.size() >= kTables) {
        // evict the least recently used entry that no captured graph references; synchronise its own device first
        for (size_t k = 0; k < tab.size(); ++k) {
            if (tab[k].pinned) continue;
            int d0 = 0;
            cudaGetDevice(&d0);
            cudaSetDevice(tab[k].dev);
            cudaDeviceSynchronize();
            cudaFree(tab[k].d);
            cudaSetDevice(d0);
            tab.erase(tab.begin() + (long)k);
            break;
        }
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
    tab.push_back({dev, h, std::vector<unsigned char>(p, p + bytes), d, pin});
    return d;
}
const int32_t* lag_table(const int32_t* lags, int64_t n, cudaStream_t s) {
    return (const int32_t*)host_table(lags, sizeof(int32_t) * (size_t)n, s);
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
