// Launch counting and per-kernel CUDA-event timing (tracing subsystem).
// When enabled, every instrumented launcher records a start/stop event pair on the stream it
// launches on; mtgr_prof_query() resolves them into per-kind launch counts and device time.
#include <cstdlib>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges reach nsys / ncu when a tool is attached

#include "common.cuh"
#include "prof.h"

namespace mtgr {

static std::atomic<long long> g_launches{0};
static std::atomic<int> g_prof_on{0};
static std::mutex g_mu;
struct Rec {
  int kind;
  cudaEvent_t a, b;
};
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_pool;
static long long g_count[PROF_NKINDS];
static double g_ms[PROF_NKINDS];

static const char* kNames[PROF_NKINDS] = {
    "gln_fwd", "gln_bwd", "gemm_qkvu", "gemm_out", "gemm_dgrad", "gemm_wgrad", "attn_diag",
    "attn_fwd", "attn_bwd_dv", "attn_bwd_dk", "attn_bwd_dq", "colsum", "other", "head", "token", "embed", "attn_bwd_scores",
    "attn_bwd_dk_fused", "attn_bwd_kv", "attn_bwd_drab"};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// MTGR_NVTX=1: every instrumented launch is wrapped in an NVTX range named by its kind (host
// timeline of the launches for nsys; ncu --nvtx filters by it)
static bool nvtx_on() {
  static const bool on = [] { const char* e = getenv("MTGR_NVTX"); return e != nullptr && e[0] == '1'; }();
  return on;
}

ProfScope::ProfScope(int kind, cudaStream_t st) : kind_(kind), st_(st), on_(false) {
  if (nvtx_on()) {
    nvtxRangePushA(kNames[kind]);
    nv_ = true;
  }
  if (g_prof_on.load(std::memory_order_relaxed)) {
    std::lock_guard<std::mutex> lk(g_mu);
    a_ = get_event();
    b_ = get_event();
    cudaEventRecord(a_, st_);
    on_ = true;
  }
}
ProfScope::~ProfScope() {
  if (on_) {
    cudaEventRecord(b_, st_);
    std::lock_guard<std::mutex> lk(g_mu);
    g_recs.push_back({kind_, a_, b_});
  }
  if (nv_) nvtxRangePop();
}

static void resolve() {
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    g_count[r.kind] += 1;
    g_ms[r.kind] += ms;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

}  // namespace mtgr

using namespace mtgr;

MTGR_API int64_t mtgr_launch_count(void) { return g_launches.load(); }

MTGR_API void mtgr_prof_enable(int32_t on) { g_prof_on.store(on ? 1 : 0); }

MTGR_API void mtgr_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  resolve();
  for (int k = 0; k < PROF_NKINDS; ++k) {
    g_count[k] = 0;
    g_ms[k] = 0.0;
  }
}

MTGR_API int32_t mtgr_prof_num_kinds(void) { return PROF_NKINDS; }

MTGR_API const char* mtgr_prof_kind_name(int32_t kind) {
  return (kind >= 0 && kind < PROF_NKINDS) ? kNames[kind] : "?";
}

MTGR_API mtgr_status_t mtgr_prof_query(int32_t kind, int64_t* launches, double* total_ms) {
  if (kind < 0 || kind >= PROF_NKINDS || !launches || !total_ms)
    return set_error(MTGR_E_ARG, "mtgr_prof_query: invalid arguments");
  std::lock_guard<std::mutex> lk(g_mu);
  resolve();
  *launches = g_count[kind];
  *total_ms = g_ms[kind];
  return MTGR_OK;
}
