// Shared device/host helpers of libmtgr (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/mtgr.h"

#define MTGR_API extern "C" __attribute__((visibility("default")))

namespace mtgr {

// ------------------------------------------------------------------ status plumbing
mtgr_status_t set_error(mtgr_status_t s, const char* fmt, ...);
mtgr_status_t check_launch(const char* what);

#define MTGR_CHECK(cond, code, ...)                                   \
  do {                                                                \
    if (!(cond)) return ::mtgr::set_error((code), __VA_ARGS__);      \
  } while (0)

#define MTGR_TRY(expr)                              \
  do {                                              \
    mtgr_status_t _s = (expr);                      \
    if (_s != MTGR_OK) return _s;                   \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// bump allocator over a caller workspace
struct Carve {
  char* base;
  size_t cap, used = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t n) {
    used = align_up(used, 256);
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += n * sizeof(T);
    return p;
  }
  bool ok() const { return used <= cap; }
};

int num_sms();

// ------------------------------------------------------------------ device math
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <class T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// silu(s) = s * sigmoid(s); precise form (expf + IEEE division) for the parity paths
__device__ __forceinline__ float silu_f(float s) { return s / (1.0f + expf(-s)); }
// silu'(s) = sigmoid(s) * (1 + s * (1 - sigmoid(s)))
__device__ __forceinline__ float dsilu_f(float s) {
  float sg = 1.0f / (1.0f + expf(-s));
  return sg * (1.0f + s * (1.0f - sg));
}

// rab bucket (R#4): min(NB-1, floor(log2(max(|dt|,1))))
__device__ __forceinline__ int rab_bucket(long long dt, int nb) {
  unsigned long long a = dt < 0 ? (unsigned long long)(-dt) : (unsigned long long)dt;
  if (a < 1) a = 1;
  int b = 63 - __clzll((long long)a);
  return b < nb - 1 ? b : nb - 1;
}

// per-user view of the jagged metadata
struct UserSpan {
  int off, L, ns, nr;
  float nu;
};
__device__ __forceinline__ UserSpan load_user(const mtgr_jagged_t& j, int u) {
  UserSpan s;
  s.off = j.offsets[u];
  s.L = j.offsets[u + 1] - s.off;
  s.ns = j.n_static[u];
  s.nr = j.n_rt[u];
  s.nu = j.inv_norm ? j.inv_norm[u] : (s.L > 0 ? 1.0f / (float)s.L : 0.f);
  return s;
}

// The dynamic-mask predicate restricted to the key range [0, ns+nr) (R#8-R#12):
// row i (reader) may read column j < ns always; columns ns <= j < ns+nr iff i >= ns and
// ts_j < ts_i.  The diagonal of non-static rows and all candidate columns (only ever visible
// to themselves, rule 3) are handled by the diagonal term, never by this predicate.
__device__ __forceinline__ bool visible_offdiag(int i, int j, int ns, long long ts_i,
                                                long long ts_j) {
  return (j < ns) || (i >= ns && ts_j < ts_i);
}

// The full mask (MTGR_MASK_FULL: Table 4's "w/o dynamic mask" read as full attention, SPEC
// S:345) restricted the same way: every static and real-time key [0, ns+nr) is visible to every
// row, except the row's own column for non-static rows (their diagonal term adds it).
__device__ __forceinline__ bool visible_offdiag_full(int i, int j, int ns, int nr) {
  return j < ns + nr && (i < ns || i != j);
}

}  // namespace mtgr
