// common.cuh -- shared device helpers of the fMoE B200 path (sm_100a).
//
// Packed top-k keys: the order "score descending, id ascending" (R5) is
// the unsigned order of a 64-bit key = (orderable(score) << 32) | (~id32):
// a larger key is a better candidate, so every merge is a plain u64 max.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace fmoe {

constexpr int kWarp = 32;
constexpr int kMaxK = 64;
constexpr int kMaxE = 64;

struct Bf16Tag {};
struct F32Tag {};

// ---------------------------------------------------------------- keys
__device__ __forceinline__ uint32_t orderable(float s) {
  s = s + 0.0f;                                  // -0.0 -> +0.0 (canonical)
  uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float from_orderable(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
// NaN never enters a top-k list: it maps to the empty key 0.
__device__ __forceinline__ uint64_t pack_key(float s, uint32_t id) {
  if (s != s) return 0ull;
  return (uint64_t(orderable(s)) << 32) | uint64_t(0xffffffffu - id);
}
__device__ __forceinline__ int64_t key_id(uint64_t key) {
  return key == 0ull ? -1ll : int64_t(0xffffffffu - uint32_t(key & 0xffffffffu));
}
__device__ __forceinline__ float key_score(uint64_t key) {
  return key == 0ull ? -__int_as_float(0x7f800000) : from_orderable(uint32_t(key >> 32));
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xffffffffu, uint32_t(v), src);
  uint32_t hi = __shfl_sync(0xffffffffu, uint32_t(v >> 32), src);
  return (uint64_t(hi) << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
  uint32_t lo = __shfl_up_sync(0xffffffffu, uint32_t(v), d);
  uint32_t hi = __shfl_up_sync(0xffffffffu, uint32_t(v >> 32), d);
  return (uint64_t(hi) << 32) | lo;
}

// ---------------------------------------------------------------- warp top-k
// A warp-distributed list sorted descending: entry j lives in lane j%32,
// register slot j/32.  KPL = ceil(kmax/32) slots.  All lanes call every method
// with warp-uniform arguments.
template <int KPL>
struct WarpTopK {
  uint64_t v[KPL];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < KPL; ++s) v[s] = 0ull;
  }
  // key at index k-1 (the current admission threshold)
  __device__ __forceinline__ uint64_t kth(int k) const {
    const int j = k - 1;
    uint64_t x = v[0];
#pragma unroll
    for (int s = 1; s < KPL; ++s)
      if (j / 32 == s) x = v[s];
    return shfl_u64(x, j & 31);
  }
  // insert key c (warp-uniform), assumed better than kth(k) and not present.
  __device__ __forceinline__ void insert(uint64_t c) {
    const int lane = threadIdx.x & 31;
    int pos = 0;
#pragma unroll
    for (int s = 0; s < KPL; ++s) pos += __popc(__ballot_sync(0xffffffffu, v[s] > c));
#pragma unroll
    for (int s = KPL - 1; s >= 0; --s) {
      uint64_t up = shfl_up_u64(v[s], 1);
      uint64_t carry = (s > 0) ? shfl_u64(v[s > 0 ? s - 1 : 0], 31) : 0ull;
      if (lane == 0) up = carry;
      const int j = s * 32 + lane;
      if (j > pos) v[s] = up;
      else if (j == pos) v[s] = c;
    }
  }
  // offer one candidate per lane (keys unique); admits those beating kth(k).
  __device__ __forceinline__ void offer(uint64_t key, int k) {
    uint64_t thr = kth(k);
    unsigned m = __ballot_sync(0xffffffffu, key > thr);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t c = shfl_u64(key, src);
      if (c > thr) {
        insert(c);
        thr = kth(k);
      }
    }
  }
  // entry j (0-based), returned on every lane
  __device__ __forceinline__ uint64_t get(int j) const {
    uint64_t x = v[0];
#pragma unroll
    for (int s = 1; s < KPL; ++s)
      if (j / 32 == s) x = v[s];
    return shfl_u64(x, j & 31);
  }
  // store entries [0, k) to dst (coalesced)
  __device__ __forceinline__ void store(uint64_t* dst, int k) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 0; s < KPL; ++s) {
      const int j = s * 32 + lane;
      if (j < k) dst[j] = v[s];
    }
  }
};

// k == 1 specialisation: each lane keeps its own best key (one max per row,
// no warp traffic); the warp maximum is formed only when read.
template <>
struct WarpTopK<0> {
  uint64_t v[1];
  __device__ __forceinline__ void init() { v[0] = 0ull; }
  __device__ __forceinline__ void offer(uint64_t key, int) { v[0] = key > v[0] ? key : v[0]; }
  __device__ __forceinline__ uint64_t get(int) const {
    uint64_t m = v[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x = shfl_u64(m, (threadIdx.x & 31) ^ o);
      m = x > m ? x : m;
    }
    return m;
  }
  __device__ __forceinline__ uint64_t kth(int) const { return get(0); }
  __device__ __forceinline__ void store(uint64_t* dst, int) const {
    const uint64_t m = get(0);
    if ((threadIdx.x & 31) == 0) dst[0] = m;
  }
};

// ---------------------------------------------------------------- bf16 / 16-byte chunks
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8], Bf16Tag) {
  f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xffff0000u);
}

template <typename Tag> struct StoreT;
template <> struct StoreT<Bf16Tag> {
  using T = __nv_bfloat16;
  static constexpr int kElemsPer16B = 8;
  static constexpr int kBytes = 2;
};
template <> struct StoreT<F32Tag> {
  using T = float;
  static constexpr int kElemsPer16B = 4;
  static constexpr int kBytes = 4;
};

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float to_store_value(float x, Bf16Tag) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
__device__ __forceinline__ float to_store_value(float x, F32Tag) { return x; }

// ---------------------------------------------------------------- mbarrier + bulk async copy (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA, non-tensor), completion counted on `bar`.
// bytes and both addresses must be multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- device phase tracer
// When a trace buffer is passed (fmoe_debug_trace, a debug entry point),
// thread 0 of every block records %globaltimer at phase boundaries:
// trace[block][phase].  Attributes a scan's time to launch, staging,
// streaming and the merge tail.
constexpr int kTraceBlocks = 4096;
constexpr int kTracePhases = 8;
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// same, from whichever single thread calls it
__device__ __forceinline__ void trace_mark_here(unsigned long long* trace, int phase) {
  if (trace && blockIdx.x < kTraceBlocks) trace[blockIdx.x * kTracePhases + phase] = globaltimer();
}
__device__ __forceinline__ void trace_mark(unsigned long long* trace, int phase) {
  if (trace && threadIdx.x == 0 && blockIdx.x < kTraceBlocks)
    trace[blockIdx.x * kTracePhases + phase] = globaltimer();
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of this library waits for the preceding grid on the stream
// before touching global memory it may depend on, and lets the next grid
// launch once its main loop is done (PDL, sm_90+).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace fmoe
