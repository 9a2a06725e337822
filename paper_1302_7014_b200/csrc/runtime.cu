// runtime.cu -- status strings, CUDA error capture, launch accounting and the
// optional per-kernel CUDA-event profiler of libpeel (peel.h "Measurement support").
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace peel {

static char g_cuda_err[512] = "";

void set_cuda_error(cudaError_t e, const char *where) {
    snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s (%s)", where, cudaGetErrorName(e),
             cudaGetErrorString(e));
}

struct ProfEntry {
    const char *name;
    cudaEvent_t a, b;
};

// the profiling tables are shared by every host thread (peel_sweep's batch workers call the
// library concurrently): every access below holds g_mu
static std::recursive_mutex g_mu;
static bool g_prof_on = false;
static std::vector<ProfEntry> g_prof;          // events of the current call
static std::vector<ProfEntry> g_pool;          // recycled events
static uint32_t g_launches = 0;
static std::vector<double> g_round_ms;                 // per-round device time of the last peel
static std::vector<const char *> g_res_names;  // resolved results of the last call
static std::vector<double> g_res_ms;
static std::vector<uint32_t> g_res_n;

static ProfEntry take_pair(const char *name) {
    ProfEntry p;
    if (!g_pool.empty()) {
        p = g_pool.back();
        g_pool.pop_back();
    } else {
        cudaEventCreate(&p.a);
        cudaEventCreate(&p.b);
    }
    p.name = name;
    return p;
}

// Launch counts and events accumulate from the first call after the last blocking
// (collecting) call, so an async iblt_insert followed by a blocking iblt_peel report
// together.
static bool g_collected = true;
static int g_hold = 0;  // > 0 inside a call made of public calls (peel_sweep): one report

void prof_hold(bool on) { std::lock_guard<std::recursive_mutex> lk(g_mu); g_hold += on ? 1 : -1; }
void prof_add_launches(uint32_t n) { std::lock_guard<std::recursive_mutex> lk(g_mu); g_launches += n; }
static bool g_capture = false;  // inside a stream capture: no events, no counts (the replay is timed)
void prof_capture(bool on) { std::lock_guard<std::recursive_mutex> lk(g_mu); g_capture = on; }

void prof_begin_call() { std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!g_collected || g_hold) return;
    g_collected = false;
    g_launches = 0;
    g_round_ms.clear();
    for (auto &p : g_prof) g_pool.push_back(p);
    g_prof.clear();
}

int prof_pre(const char *name, cudaStream_t s) { std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!g_prof_on || g_capture) return -1;
    ProfEntry p = take_pair(name);
    cudaEventRecord(p.a, s);
    g_prof.push_back(p);
    return (int)g_prof.size() - 1;
}

// the entry index (not "the last entry"): concurrent threads interleave their entries
void prof_post(int entry, cudaStream_t s) { std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (g_capture) return;
    g_launches++;
    if (!g_prof_on || entry < 0 || entry >= (int)g_prof.size()) return;
    cudaEventRecord(g_prof[entry].b, s);
}

int prof_collect() { std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (g_hold) return 0;
    g_collected = true;
    g_res_names.clear();
    g_res_ms.clear();
    g_res_n.clear();
    if (!g_prof_on) return 0;
    for (auto &p : g_prof) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) != cudaSuccess) ms = -1.f;
        size_t i = 0;
        for (; i < g_res_names.size(); i++)
            if (strcmp(g_res_names[i], p.name) == 0) break;
        if (i == g_res_names.size()) {
            g_res_names.push_back(p.name);
            g_res_ms.push_back(0.0);
            g_res_n.push_back(0);
        }
        g_res_ms[i] += ms;
        g_res_n[i] += 1;
    }
    return (int)g_res_names.size();
}

bool prof_enabled() { return g_prof_on; }
void prof_set_rounds(const std::vector<double> &ms) { std::lock_guard<std::recursive_mutex> lk(g_mu); g_round_ms = ms; }

cudaError_t raise_smem(const void *kern, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> cur;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t &c = cur[std::make_pair(dev, kern)];
    if (bytes <= c) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c = bytes;
    return e;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace peel

extern "C" {

const char *peel_strerror(int s) {
    switch (s) {
        case PEEL_OK: return "PEEL_OK";
        case PEEL_EINVAL: return "PEEL_EINVAL: invalid argument or input";
        case PEEL_ENOMEM: return "PEEL_ENOMEM: workspace too small or allocation failed";
        case PEEL_ECUDA: return "PEEL_ECUDA: CUDA runtime error";
        case PEEL_ETRUNC: return "PEEL_ETRUNC: more rounds/keys than the caller's capacity";
        case PEEL_ENCCL: return "PEEL_ENCCL: NCCL error";
        case PEEL_EOVERFLOW: return "PEEL_EOVERFLOW: packed state overflow; use PEEL_FLAG_CSR";
        case PEEL_EPEER: return "PEEL_EPEER: another rank of the communicator failed";
        default: return "unknown peel_status";
    }
}

const char *peel_last_cuda_error(void) { return peel::g_cuda_err; }

int peel_abi_version(void) { return PEEL_ABI_VERSION; }

void peel_profile_enable(int on) { peel::g_prof_on = on != 0; }

int peel_profile_read(const char **names, double *ms, uint32_t *launches, int cap) {
    int n = (int)peel::g_res_names.size();
    for (int i = 0; i < n && i < cap; i++) {
        if (names) names[i] = peel::g_res_names[i];
        if (ms) ms[i] = peel::g_res_ms[i];
        if (launches) launches[i] = peel::g_res_n[i];
    }
    return n;
}

uint32_t peel_last_launches(void) { return peel::g_launches; }

int peel_profile_rounds(double *ms, uint32_t cap) {
    int n = (int)peel::g_round_ms.size();
    for (int i = 0; i < n && i < (int)cap; i++) ms[i] = peel::g_round_ms[i];
    return n;
}

}  // extern "C"
