// Dynamic hash embedding table and the ID-unique step of the embedding lookup (
// PAPER.md §5 "Dynamic Hash Table" and "Embedding Lookup").
//
//   "We employ a decoupled architecture for hash table, which separates key and value storage
//    into distinct structures.  The key structure maintains a lightweight mapping table
//    containing keys and corresponding pointers to embedding vectors, while the value structure
//    stores both the embedding vectors and auxiliary metadata (e.g., counters and timestamps)
//    required for eviction policies".  Expansion replicates only the key structure.
//   "two-stage ID unique operation to reduce redundant IDs before and after ID communication"
//    (P:355).
//
// Key structure: open addressing with linear probing over a power-of-two bucket array of
// (int64 key, int32 slot); EMPTY / TOMBSTONE sentinels.  A missing key is claimed with a 64-bit
// CAS; the claiming thread allocates a value slot (free stack first, then the bump pointer),
// initialises the row from a counter-based hash of (seed, key, column) and publishes the slot;
// concurrent readers of a claimed bucket wait for the slot.  Value structure: rows [cap_v][dim]
// fp32, per-slot access counter, last-access timestamp and owning key (for eviction).
// Unique: the same probing scheme on a scratch set; the unique index of a key is taken from an
// atomic counter by its first inserter (the order of the unique list is unspecified; the
// inverse map is exact).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {
namespace {

constexpr long long KEY_EMPTY = (long long)0x8000000000000000ull;  // INT64_MIN
constexpr long long KEY_TOMB = KEY_EMPTY + 1;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// initial value of column c of key k: init_scale * U(-1, 1) from mix64(seed ^ mix64(k) + c)
__device__ __forceinline__ float init_value(uint64_t seed, long long k, int c, float scale) {
  const uint64_t h = mix64(seed ^ (mix64((uint64_t)k) + (uint64_t)c));
  const float u = (float)(h >> 40) * (1.0f / 16777216.0f);  // [0, 1), 24 bits
  return scale * (2.0f * u - 1.0f);
}

__global__ void hash_init_kernel(mtgr_hash_table_t t) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < t.cap_k; b += (int64_t)gridDim.x * blockDim.x) {
    t.keys[b] = KEY_EMPTY;
    t.slots[b] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { t.alloc[0] = 0; t.alloc[1] = 0; t.alloc[2] = 0; }
}

__device__ int alloc_slot(const mtgr_hash_table_t& t) {
  // recycled slots first (evicted keys), then fresh ones
  int top = atomicSub(&t.alloc[1], 1);
  if (top > 0) return t.free_stack[top - 1];
  atomicAdd(&t.alloc[1], 1);  // undo (stack was empty)
  const int s = atomicAdd(&t.alloc[0], 1);
  return (int64_t)s < t.cap_v ? s : -2;
}

// thread per key: probe; a missing key is claimed with a CAS, the claiming thread allocates a
// slot, initialises the row and publishes the slot (threads meeting a claimed bucket wait for
// the publication; independent thread scheduling lets a waiting lane and the claiming lane of
// the same warp both progress)
__global__ void hash_find_or_insert_kernel(mtgr_hash_table_t t, const long long* __restrict__ ids, int n,
                                           long long now, int insert, int* __restrict__ out_slots) {
  const uint64_t mask = (uint64_t)t.cap_k - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long k = ids[i];
    int slot = -1;
    bool claimed = false;
    uint64_t b = mix64((uint64_t)k) & mask;
    for (int64_t probe = 0; probe < t.cap_k; ++probe, b = (b + 1) & mask) {
      long long cur = *reinterpret_cast<volatile long long*>(&t.keys[b]);
      if (cur == KEY_EMPTY) {
        if (!insert) break;
        cur = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&t.keys[b]),
                                   (unsigned long long)KEY_EMPTY, (unsigned long long)k);
        if (cur == KEY_EMPTY) {
          slot = alloc_slot(t);
          claimed = true;
          break;
        }
      }
      if (cur == k) {  // present (possibly being published)
        int s;
        while ((s = *reinterpret_cast<volatile int*>(&t.slots[b])) == -1) {
        }
        slot = s;
        break;
      }
      // another key or a tombstone: keep probing
    }
    if (claimed) {
      if (slot >= 0) {
        t.slot_key[slot] = k;
        float* row = t.values + (int64_t)slot * t.dim;
        for (int c = 0; c < t.dim; ++c) row[c] = init_value(t.seed, k, c, t.init_scale);
        t.counter[slot] = 0;
        __threadfence();
      } else {
        atomicAdd(&t.alloc[2], 1);  // value structure full: counted failure
      }
      *reinterpret_cast<volatile int*>(&t.slots[b]) = slot;  // publish
    }
    if (slot >= 0) {
      atomicAdd(&t.counter[slot], 1u);
      t.ts[slot] = now;
    }
    out_slots[i] = slot;
  }
}

// Row kernels map one thread to one (row, column) element: rows are narrow (16-32 values), so
// a warp per row would leave most lanes idle; consecutive threads walk a row, then the next.
template <class T>
__global__ void hash_gather_kernel(mtgr_hash_table_t t, const int* __restrict__ slots, int n, T* __restrict__ out) {
  const int64_t total = (int64_t)n * t.dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / t.dim;
    const int c = (int)(e - i * t.dim);
    const int s = slots[i];
    out[e] = from_f<T>(s < 0 ? 0.f : t.values[(int64_t)s * t.dim + c]);
  }
}

// values[slot] -= lr * grad (atomics: duplicate slots accumulate)
template <class T>
__global__ void hash_sgd_kernel(mtgr_hash_table_t t, const int* __restrict__ slots, int n,
                                const T* __restrict__ g, float lr) {
  const int64_t total = (int64_t)n * t.dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / t.dim;
    const int c = (int)(e - i * t.dim);
    const int s = slots[i];
    if (s >= 0) atomicAdd(t.values + (int64_t)s * t.dim + c, -lr * to_f(g[e]));
  }
}

// eviction by last-access time: the key bucket becomes a tombstone, the slot returns to the
// free stack
__global__ void hash_evict_kernel(mtgr_hash_table_t t, long long ts_before) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < t.cap_k; b += (int64_t)gridDim.x * blockDim.x) {
    const long long k = t.keys[b];
    if (k == KEY_EMPTY || k == KEY_TOMB) continue;
    const int s = t.slots[b];
    if (s >= 0 && t.ts[s] < ts_before) {
      t.keys[b] = KEY_TOMB;
      t.slots[b] = -1;
      const int top = atomicAdd(&t.alloc[1], 1);
      t.free_stack[top] = s;
      t.slot_key[s] = KEY_EMPTY;
    }
  }
}

// expansion: re-insert every live (key, slot) of the old key structure into the new one (the
// value structure is untouched)
__global__ void hash_rehash_kernel(const long long* __restrict__ okeys, const int* __restrict__ oslots,
                                   int64_t ocap, long long* nkeys, int* nslots, int64_t ncap) {
  const uint64_t mask = (uint64_t)ncap - 1;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < ocap; b += (int64_t)gridDim.x * blockDim.x) {
    const long long k = okeys[b];
    if (k == KEY_EMPTY || k == KEY_TOMB) continue;
    uint64_t h = mix64((uint64_t)k) & mask;
    for (;;) {
      const long long cur = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&nkeys[h]),
                                                 (unsigned long long)KEY_EMPTY, (unsigned long long)k);
      if (cur == KEY_EMPTY) { nslots[h] = oslots[b]; break; }
      h = (h + 1) & mask;
    }
  }
}

__global__ void fill_kernel(long long* keys, int* vals, int64_t n) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    keys[b] = KEY_EMPTY;
    vals[b] = -1;
  }
}

// unique: scratch set of cap buckets (keys, index); count[0] = number of unique ids
__global__ void unique_kernel(const long long* __restrict__ ids, int n, long long* skeys, int* sidx, int64_t cap,
                              int* count, long long* uniq, int* inverse) {
  const uint64_t mask = (uint64_t)cap - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long k = ids[i];
    uint64_t b = mix64((uint64_t)k) & mask;
    int idx = -1;
    for (;;) {
      long long cur = *reinterpret_cast<volatile long long*>(&skeys[b]);
      if (cur == KEY_EMPTY) {
        cur = (long long)atomicCAS(reinterpret_cast<unsigned long long*>(&skeys[b]),
                                   (unsigned long long)KEY_EMPTY, (unsigned long long)k);
        if (cur == KEY_EMPTY) {
          idx = atomicAdd(count, 1);
          uniq[idx] = k;
          __threadfence();
          *reinterpret_cast<volatile int*>(&sidx[b]) = idx;
          break;
        }
      }
      if (cur == k) {
        while ((idx = *reinterpret_cast<volatile int*>(&sidx[b])) == -1) {
        }
        break;
      }
      b = (b + 1) & mask;
    }
    inverse[i] = idx;
  }
}

// segment sums by an index map: out[inverse[i]] += g[i] (rows of dim); out zeroed by the caller
template <class T>
__global__ void segsum_kernel(const T* __restrict__ g, const int* __restrict__ inverse, int n, int dim,
                              float* __restrict__ out) {
  const int64_t total = (int64_t)n * dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / dim;
    const int c = (int)(e - i * dim);
    atomicAdd(out + (int64_t)inverse[i] * dim + c, to_f(g[e]));
  }
}

// the same sums with per-block privatisation of the first `hot` unique rows in shared memory:
// the unique index of an ID is its first-arrival order, so the hottest IDs of a Zipf stream
// (which appear early) get small indices, and their many occurrences accumulate in shared
// memory instead of serialising on the same global addresses; each block then adds its partial
// rows once.  Blocks own contiguous row ranges.
template <class T>
__global__ void segsum_priv_kernel(const T* __restrict__ g, const int* __restrict__ inverse, int n, int dim,
                                   int hot, float* __restrict__ out) {
  extern __shared__ float acc[];  // [hot][dim]
  for (int e = threadIdx.x; e < hot * dim; e += blockDim.x) acc[e] = 0.f;
  __syncthreads();
  const int64_t rows_per = ((int64_t)n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per, r1 = min((int64_t)n, r0 + rows_per);
  for (int64_t e = r0 * dim + threadIdx.x; e < r1 * dim; e += blockDim.x) {
    const int64_t i = e / dim;
    const int c = (int)(e - i * dim);
    const int key = inverse[i];
    const float v = to_f(g[e]);
    if (key < hot) atomicAdd(&acc[key * dim + c], v);
    else atomicAdd(out + (int64_t)key * dim + c, v);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < hot * dim; e += blockDim.x)
    if (acc[e] != 0.f) atomicAdd(out + e, acc[e]);
}

// row moves, 16 bytes per thread when the row allows it (else one element):
//   gather (PUT = 0): out[i] = src[idx[i]];   scatter (PUT = 1): out[idx[i]] = src[i]
template <class V, int PUT>
__global__ void move_rows_kernel(const V* __restrict__ src, const int* __restrict__ idx, int n, int vpr,
                                 V* __restrict__ out) {
  const int64_t total = (int64_t)n * vpr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / vpr;
    const int c = (int)(e - i * vpr);
    const int64_t j = idx[i];
    if (PUT) out[j * vpr + c] = src[e];
    else out[e] = src[j * vpr + c];
  }
}

template <int PUT>
mtgr_status_t move_rows(const void* src, const int32_t* idx, int32_t n, int64_t row_bytes, void* out,
                        cudaStream_t st);

// owner partition for the all-to-all: dest(k) = mix64(k ^ salt) % world; per-destination counts
// and each id's position in the destination-grouped send buffer (order within a destination:
// by atomic arrival, unspecified)
__global__ void partition_count_kernel(const long long* __restrict__ ids, int n, int world, uint64_t salt,
                                       int* counts, int* dest) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = (int)(mix64((uint64_t)ids[i] ^ salt) % (uint64_t)world);
    dest[i] = r;
    atomicAdd(&counts[r], 1);
  }
}
__global__ void partition_place_kernel(const long long* __restrict__ ids, int n, const int* __restrict__ dest,
                                       const int* __restrict__ starts, int* fill, long long* send, int* pos) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = dest[i];
    const int p = starts[r] + atomicAdd(&fill[r], 1);
    send[p] = ids[i];
    pos[i] = p;
  }
}

__global__ void scan_small_kernel(const int* counts, int n, int* starts) {
  int acc = 0;
  for (int i = 0; i < n; ++i) { starts[i] = acc; acc += counts[i]; }
}

int grid_for(int64_t work_items, int per_block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div64(work_items, per_block), 16 * 148));
}

template <int PUT>
mtgr_status_t move_rows(const void* src, const int32_t* idx, int32_t n, int64_t row_bytes, void* out,
                        cudaStream_t st) {
  if (row_bytes % 16 == 0) {
    const int vpr = (int)(row_bytes / 16);
    move_rows_kernel<uint4, PUT><<<grid_for((int64_t)n * vpr, 256), 256, 0, st>>>(
        (const uint4*)src, idx, n, vpr, (uint4*)out);
  } else {
    const int vpr = (int)(row_bytes / 2);
    move_rows_kernel<uint16_t, PUT><<<grid_for((int64_t)n * vpr, 256), 256, 0, st>>>(
        (const uint16_t*)src, idx, n, vpr, (uint16_t*)out);
  }
  return check_launch(PUT ? "put_rows" : "take_rows");
}

mtgr_status_t check_table(const mtgr_hash_table_t* t) {
  MTGR_CHECK(t && t->keys && t->slots && t->values && t->counter && t->ts && t->slot_key && t->alloc &&
                 t->free_stack,
             MTGR_E_ARG, "hash table: null pointer");
  MTGR_CHECK(t->cap_k > 0 && (t->cap_k & (t->cap_k - 1)) == 0, MTGR_E_ARG, "hash table: cap_k must be a power of two");
  MTGR_CHECK(t->cap_v > 0 && t->cap_v < (1ll << 31) && t->dim > 0, MTGR_E_ARG, "hash table: bad cap_v / dim");
  return MTGR_OK;
}

}  // namespace
}  // namespace mtgr

using namespace mtgr;

MTGR_API mtgr_status_t mtgr_hash_init(const mtgr_hash_table_t* t, mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  ProfScope ps(PROF_EMBED, (cudaStream_t)stream);
  hash_init_kernel<<<grid_for(t->cap_k, 256), 256, 0, (cudaStream_t)stream>>>(*t);
  return check_launch("hash_init");
}

MTGR_API mtgr_status_t mtgr_hash_find_or_insert(const mtgr_hash_table_t* t, const int64_t* ids, int32_t n,
                                                int64_t now, int32_t insert, int32_t* slots,
                                                mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  MTGR_CHECK(n >= 0 && (n == 0 || (ids && slots)), MTGR_E_ARG, "hash_find_or_insert: bad ids / slots");
  if (n == 0) return MTGR_OK;
  ProfScope ps(PROF_EMBED, (cudaStream_t)stream);
  hash_find_or_insert_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      *t, (const long long*)ids, n, (long long)now, insert ? 1 : 0, slots);
  return check_launch("hash_find_or_insert");
}

MTGR_API mtgr_status_t mtgr_hash_gather(const mtgr_hash_table_t* t, const int32_t* slots, int32_t n,
                                        mtgr_dtype_t dtype, void* out, mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  MTGR_CHECK(n >= 0 && (n == 0 || (slots && out)), MTGR_E_ARG, "hash_gather: bad pointers");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "hash_gather: dtype");
  if (n == 0) return MTGR_OK;
  ProfScope ps(PROF_EMBED, (cudaStream_t)stream);
  const int g = grid_for((int64_t)n * t->dim, 256);
  if (dtype == MTGR_BF16)
    hash_gather_kernel<__nv_bfloat16><<<g, 256, 0, (cudaStream_t)stream>>>(*t, slots, n, (__nv_bfloat16*)out);
  else
    hash_gather_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>(*t, slots, n, (float*)out);
  return check_launch("hash_gather");
}

MTGR_API mtgr_status_t mtgr_hash_sgd(const mtgr_hash_table_t* t, const int32_t* slots, int32_t n,
                                     mtgr_dtype_t dtype, const void* grads, float lr, mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  MTGR_CHECK(n >= 0 && (n == 0 || (slots && grads)), MTGR_E_ARG, "hash_sgd: bad pointers");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "hash_sgd: dtype");
  if (n == 0) return MTGR_OK;
  ProfScope ps(PROF_EMBED, (cudaStream_t)stream);
  const int g = grid_for((int64_t)n * t->dim, 256);
  if (dtype == MTGR_BF16)
    hash_sgd_kernel<__nv_bfloat16><<<g, 256, 0, (cudaStream_t)stream>>>(*t, slots, n, (const __nv_bfloat16*)grads, lr);
  else
    hash_sgd_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>(*t, slots, n, (const float*)grads, lr);
  return check_launch("hash_sgd");
}

MTGR_API mtgr_status_t mtgr_hash_evict(const mtgr_hash_table_t* t, int64_t ts_before, mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  ProfScope ps(PROF_EMBED, (cudaStream_t)stream);
  hash_evict_kernel<<<grid_for(t->cap_k, 256), 256, 0, (cudaStream_t)stream>>>(*t, (long long)ts_before);
  return check_launch("hash_evict");
}

MTGR_API mtgr_status_t mtgr_hash_expand(const mtgr_hash_table_t* t, int64_t* new_keys, int32_t* new_slots,
                                        int64_t new_cap_k, mtgr_stream_t stream) {
  MTGR_TRY(check_table(t));
  MTGR_CHECK(new_keys && new_slots && new_cap_k >= t->cap_k && (new_cap_k & (new_cap_k - 1)) == 0, MTGR_E_ARG,
             "hash_expand: new_cap_k must be a power of two >= cap_k");
  cudaStream_t st = (cudaStream_t)stream;
  ProfScope ps(PROF_EMBED, st);
  fill_kernel<<<grid_for(new_cap_k, 256), 256, 0, st>>>((long long*)new_keys, new_slots, new_cap_k);
  MTGR_TRY(check_launch("hash_expand_fill"));
  hash_rehash_kernel<<<grid_for(t->cap_k, 256), 256, 0, st>>>((const long long*)t->keys, t->slots, t->cap_k,
                                                                (long long*)new_keys, new_slots, new_cap_k);
  return check_launch("hash_rehash");
}

MTGR_API size_t mtgr_unique_workspace_bytes(int32_t n) {
  int64_t cap = 64;
  while (cap < 2 * (int64_t)std::max(n, 1)) cap <<= 1;
  return align_up((size_t)cap * 8, 256) + align_up((size_t)cap * 4, 256) + 256;
}

MTGR_API mtgr_status_t mtgr_unique(const int64_t* ids, int32_t n, int64_t* uniq, int32_t* inverse,
                                   int32_t* count, void* ws, size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_CHECK(n >= 0 && count && (n == 0 || (ids && uniq && inverse)), MTGR_E_ARG, "unique: bad pointers");
  MTGR_CHECK(ws && ws_bytes >= mtgr_unique_workspace_bytes(n), MTGR_E_WORKSPACE, "unique: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(count, 0, sizeof(int32_t), st);
  if (n == 0) return MTGR_OK;
  int64_t cap = 64;
  while (cap < 2 * (int64_t)n) cap <<= 1;
  char* w = (char*)ws;
  long long* skeys = (long long*)w;
  int* sidx = (int*)(w + align_up((size_t)cap * 8, 256));
  ProfScope ps(PROF_EMBED, st);
  fill_kernel<<<grid_for(cap, 256), 256, 0, st>>>(skeys, sidx, cap);
  MTGR_TRY(check_launch("unique_fill"));
  unique_kernel<<<grid_for(n, 256), 256, 0, st>>>((const long long*)ids, n, skeys, sidx, cap, count,
                                                  (long long*)uniq, inverse);
  return check_launch("unique");
}

MTGR_API mtgr_status_t mtgr_segment_sum(mtgr_dtype_t dtype, const void* g, const int32_t* inverse, int32_t n,
                                        int32_t dim, float* out, int32_t n_out, mtgr_stream_t stream) {
  MTGR_CHECK(n >= 0 && dim > 0 && n_out >= 0 && out && (n == 0 || (g && inverse)), MTGR_E_ARG, "segment_sum: bad args");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "segment_sum: dtype");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(out, 0, sizeof(float) * (size_t)n_out * dim, st);
  if (n == 0) return MTGR_OK;
  ProfScope ps(PROF_EMBED, st);
  // privatise the first `hot` unique rows per block (16 KB of shared memory); 8 blocks per SM,
  // each over a contiguous range of rows so its flush is amortised
  if (n >= 2 * n_out && dim <= 128) {  // many occurrences per row (stage 1 of a skewed stream)
    const int hot = std::min(n_out, std::max(1, 4096 / dim));  // 16 KB of shared memory
    const int gr = std::max(1, std::min(ceil_div(n, 32), 8 * 148));
    const size_t sm = (size_t)hot * dim * sizeof(float);
    if (dtype == MTGR_BF16)
      segsum_priv_kernel<__nv_bfloat16><<<gr, 256, sm, st>>>((const __nv_bfloat16*)g, inverse, n, dim, hot, out);
    else
      segsum_priv_kernel<float><<<gr, 256, sm, st>>>((const float*)g, inverse, n, dim, hot, out);
  } else {
    const int gr = grid_for((int64_t)n * dim, 256);
    if (dtype == MTGR_BF16) segsum_kernel<__nv_bfloat16><<<gr, 256, 0, st>>>((const __nv_bfloat16*)g, inverse, n, dim, out);
    else segsum_kernel<float><<<gr, 256, 0, st>>>((const float*)g, inverse, n, dim, out);
  }
  return check_launch("segment_sum");
}

MTGR_API mtgr_status_t mtgr_take_rows(mtgr_dtype_t dtype, const void* src, const int32_t* idx, int32_t n,
                                      int32_t dim, void* out, mtgr_stream_t stream) {
  MTGR_CHECK(n >= 0 && dim > 0 && (n == 0 || (src && idx && out)), MTGR_E_ARG, "take_rows: bad args");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "take_rows: dtype");
  if (n == 0) return MTGR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ProfScope ps(PROF_EMBED, st);
  return move_rows<0>(src, idx, n, (int64_t)dim * (dtype == MTGR_BF16 ? 2 : 4), out, st);
}

MTGR_API mtgr_status_t mtgr_put_rows(mtgr_dtype_t dtype, const void* src, const int32_t* idx, int32_t n,
                                     int32_t dim, void* out, mtgr_stream_t stream) {
  MTGR_CHECK(n >= 0 && dim > 0 && (n == 0 || (src && idx && out)), MTGR_E_ARG, "put_rows: bad args");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "put_rows: dtype");
  if (n == 0) return MTGR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ProfScope ps(PROF_EMBED, st);
  return move_rows<1>(src, idx, n, (int64_t)dim * (dtype == MTGR_BF16 ? 2 : 4), out, st);
}

MTGR_API mtgr_status_t mtgr_partition_ids(const int64_t* ids, int32_t n, int32_t world, uint64_t salt,
                                          int32_t* counts, int32_t* dest, int32_t* starts_ws,
                                          int64_t* send, int32_t* pos, mtgr_stream_t stream) {
  MTGR_CHECK(world >= 1 && n >= 0 && counts && starts_ws && (n == 0 || (ids && dest && send && pos)), MTGR_E_ARG,
             "partition_ids: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * world, st);
  cudaMemsetAsync(starts_ws, 0, sizeof(int32_t) * 2 * world, st);
  if (n == 0) return MTGR_OK;
  ProfScope ps(PROF_EMBED, st);
  partition_count_kernel<<<grid_for(n, 256), 256, 0, st>>>((const long long*)ids, n, world, salt, counts, dest);
  MTGR_TRY(check_launch("partition_count"));
  // starts = exclusive scan of counts (starts_ws[0..world)), fill counters (starts_ws[world..2world))
  scan_small_kernel<<<1, 1, 0, st>>>(counts, world, starts_ws);  // world is small
  partition_place_kernel<<<grid_for(n, 256), 256, 0, st>>>((const long long*)ids, n, dest, starts_ws,
                                                           starts_ws + world, (long long*)send, pos);
  return check_launch("partition_place");
}
