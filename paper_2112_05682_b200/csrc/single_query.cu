// single_query.cu — the paper's O(1)-memory single-query attention (made
// stable by the running max of PAPER.md:85-90), split over key ranges (split-K), with the
// merge of the per-range states by Figure 1's global-max rescale done in
// the SAME launch by the last CTA of each group to finish (arrival ticket): one kernel per call.
//
// HBM-bound: every key costs 4*d bytes (k and v rows, bf16) and 4*d flops, 1 flop/byte.
// bf16 kernel: 8 (d = 64) or 16 (d = 128) lanes share one key row (16 B = 8 bf16 each,
// 128-bit streaming loads), the dot product finishes with xor-shuffles inside the lane group,
// and each group runs its own stream state (m*, s*, v*[8 dims per lane]) with one rescale per
// 4 keys (block max first). A CTA covers one key range of HC heads of one batch element: the
// HC rows of a key are adjacent in [B, n_k, H, d], so a warp-load of HC >= 2 heads is one
// contiguous 256-byte (or longer) run instead of head-strided 128-byte rows. Groups, warps and
// splits are merged with the same rescale rule.
//
// Partial records (workspace, float32): rec[(bh * splits + split) * (d + 2) + {0: m*, 1: s*,
// 2..: v*}], m* in log2 units of the scaled score (p = 2^(s*c - m*), c = scale*log2 e). After
// the records: per CTA group (b, head block) a 64-bit arrival ticket (counter_take: the merging
// CTA leaves it reset for the next call; uninitialised workspace is recognised and restarted by
// the first arrivals): no memset, no extra launch.
#include <cuda_bf16.h>

#include <atomic>
#include <chrono>
#include <cmath>

#include "internal.h"
#include "ptx.cuh"

namespace mea {

// experiment knobs (mea_debug_set_option), defaults = the shipped configuration
int g_sq_heads_per_cta = 0;   // 0 = automatic
int g_sq_ctas_per_sm = 0;     // 0 = automatic
int g_sq_l2_256 = 1;          // L2::256B prefetch hint on the K/V loads
int g_sq_static_pct = -1;     // keys in static per-CTA ranges (%), the rest a dynamic pool (-1: auto)

#ifdef MEA_SQ_TIMING
// timeline probe build only: per CTA {start, streaming done, record written, merge done, ticket
// taken (merging CTA), merge loads done, merge combined} (ns)
__device__ unsigned long long g_sq_times[8192][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SQ_T(i) \
  if (threadIdx.x == 0) g_sq_times[(blockIdx.y * gridDim.x + blockIdx.x) & 8191][i] = gtimer();
#else
#define SQ_T(i)
#endif

namespace {

constexpr int kSqThreads = 512;
constexpr int kSqWarps = kSqThreads / 32;
template <int D> struct SqCfg {
  static constexpr int LPR = D / 8;     // lanes per key row
  static constexpr int G = 32 / LPR;    // key groups per warp
  static constexpr int NG = kSqWarps * G;
};
constexpr int kUnroll = 2;  // warp steps in flight

struct State {
  float m, l, a[8];
};

// Merge state o into s (both relative to their own reference max, log2 units).
__device__ __forceinline__ void merge_state(State& s, const State& o) {
  const float M = fmaxf(s.m, o.m);
  if (M == -INFINITY) return;
  const float ws = ex2_approx(s.m - M), wo = ex2_approx(o.m - M);
  s.l = s.l * ws + o.l * wo;
#pragma unroll
  for (int i = 0; i < 8; ++i) s.a[i] = s.a[i] * ws + o.a[i] * wo;
  s.m = M;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <bool kL2Hint>
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  if (kL2Hint)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  return r;
}

// Final merge of one CTA group (HC heads x `splits` records each), run by the last CTA:
//   M = max_s m_s;  out = sum_s 2^(m_s - M) v*_s / sum_s 2^(m_s - M) s*_s
// Threads own (head, feature) outputs; with fewer outputs than threads the splits are divided
// among T thread subsets, each folding its splits with the online rule, then combined in smem.
template <int NT>
__device__ void merge_group(const SqParams& p, const float* __restrict__ rec, int bh0, int HC, int d, float* smem) {
  const int O = HC * d;
  const int T = O >= NT ? 1 : NT / O;
  const int splits = p.splits;
  float* sm_m = smem;                 // [T][O]
  float* sm_l = sm_m + T * O;
  float* sm_a = sm_l + T * O;
  for (int t = threadIdx.x; t < O * T; t += NT) {
    const int o = t % O, j = t / O;
    const int hl = o / d, f = o % d;
    const float* base = rec + (size_t)(bh0 + hl) * splits * (d + 2);
    float m = -INFINITY, l = 0.f, a = 0.f;
    constexpr int U = 20;   // 148 splits over 8 thread subsets: one batch of independent loads
    for (int s0 = j; s0 < splits; s0 += U * T) {
      float ms[U], ls[U], as[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * T;
        const bool ok = s < splits;
        const float* r = base + (size_t)(ok ? s : 0) * (d + 2);
        ms[u] = ok ? __ldcg(r) : -INFINITY;
        ls[u] = ok ? __ldcg(r + 1) : 0.f;
        as[u] = ok ? __ldcg(r + 2 + f) : 0.f;
      }
      float M = m;
#pragma unroll
      for (int u = 0; u < U; ++u) M = fmaxf(M, ms[u]);
      if (M == -INFINITY) continue;
      const float w0 = ex2_approx(m - M);
      l *= w0;
      a *= w0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float w = ex2_approx(ms[u] - M);
        l = fmaf(w, ls[u], l);
        a = fmaf(w, as[u], a);
      }
      m = M;
    }
    sm_m[j * O + o] = m;
    sm_l[j * O + o] = l;
    sm_a[j * O + o] = a;
  }
  SQ_T(5)
  __syncthreads();
  for (int o = threadIdx.x; o < O; o += NT) {
    float M = -INFINITY;
    for (int j = 0; j < T; ++j) M = fmaxf(M, sm_m[j * O + o]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY)
      for (int j = 0; j < T; ++j) {
        const float w = ex2_approx(sm_m[j * O + o] - M);
        L = fmaf(w, sm_l[j * O + o], L);
        A = fmaf(w, sm_a[j * O + o], A);
      }
    const int hl = o / d, f = o % d;
    const size_t bh = (size_t)(bh0 + hl);
    if (p.mode == 0) {
      const float r = A / L;
      if (p.out_f32) static_cast<float*>(p.out)[bh * d + f] = r;
      else static_cast<__nv_bfloat16*>(p.out)[bh * d + f] = __float2bfloat16_rn(r);
    } else {  // the merged triple, m in natural-log units, for the cross-GPU merge
      if (f == 0) {
        p.tri_m[bh * p.tri_ms_stride] = M * 0.6931471805599453f;
        p.tri_s[bh * p.tri_ms_stride] = L;
      }
      p.tri_v[bh * p.tri_v_stride + f] = A;
    }
  }
}

// The arrival ticket of a CTA group in the workspace is a 64-bit word (kClean << 24 | count).
// The CTA that merges a group resets it to (kClean, 0) at the
// end of the call, so the next call on the same workspace counts from 0 with plain atomicAdds.
// A word with another tag (uninitialised workspace, first use) is stale: its first users' adds
// are void and they race to replace it by (kClean, 1) with CAS, retrying on the value that beat
// them (no further adds, so the race ends once the first users stop); a user that finds the word
// already restarted counts itself in with a fresh add. Returns the 0-based count this user took.
constexpr unsigned long long kClean = 0xC1EA5ED5A1ull;   // 40-bit marker of a reset counter
// completes a take whose first atomicAdd returned `old`
__device__ __noinline__ unsigned counter_take_slow(unsigned long long* t, unsigned long long old) {
  unsigned long long cur = old + 1;
  while (true) {
    if ((cur >> 24) == kClean) {  // restarted by another user: count in on the fresh word
      old = atomicAdd(t, 1ull);
      if ((old >> 24) == kClean) return (unsigned)(old & 0xFFFFFFull);
      cur = old + 1;
      continue;
    }
    const unsigned long long prev = atomicCAS(t, cur, (kClean << 24) | 1ull);
    if (prev == cur) return 0u;
    cur = prev;
  }
}
__device__ __forceinline__ unsigned counter_finish(unsigned long long* t, unsigned long long old) {
  if ((old >> 24) == kClean) return (unsigned)(old & 0xFFFFFFull);
  return counter_take_slow(t, old);
}
__device__ __forceinline__ unsigned counter_take(unsigned long long* t) {
  return counter_finish(t, atomicAdd(t, 1ull));
}

// Counts this CTA in (its records are written); the LAST of the group's `splits` CTAs merges and
// resets the group's ticket for the next call.
template <int NT>
__device__ __forceinline__ void finish_cta(const SqParams& p, int group, int bh0, int HC, int d, float* smem) {
  __shared__ int s_last;
  // release: the CTA's record writes (ordered before thread 0 by the barrier) become visible
  // device-wide before the ticket counts them (fence.acq_rel is cumulative); acquire on the
  // last arrival before anyone reads the other CTAs' records
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    const bool last = counter_take(p.tickets + group) + 1 == (unsigned)p.splits;
    if (last) fence_acq_rel_gpu();
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  SQ_T(4)
  merge_group<NT>(p, p.rec, bh0, HC, d, smem);
  if (threadIdx.x == 0) {   // every CTA of the group has arrived (and made its last claim)
    p.tickets[group] = kClean << 24;
    if (p.claims) p.claims[group] = kClean << 24;
  }
  SQ_T(3)
}

template <int D, int HC, bool kL2Hint>
__global__ void __launch_bounds__(kSqThreads) sq_bf16_kernel(const SqParams p) {
  using C = SqCfg<D>;
  constexpr int LPR = C::LPR, G = C::G, NG = C::NG;
  constexpr int KS = NG / HC;                 // key slots per CTA step (groups per head)
  constexpr int kStep = 4 * KS;               // keys per CTA step (4 per group)
  const int split = blockIdx.x, group = blockIdx.y;
  const int hb = p.H / HC;                    // head blocks per batch element
  const int b = group / hb, h0 = (group % hb) * HC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, cidx = lane % LPR;
  const int gid = warp * G + g;               // group in the CTA
  const int hl = gid % HC, ks = gid / HC;     // its head (of the block) and key slot
  const int n_k = p.n_k;
  // static range of this split; with a pool, the keys past splits * static_keys are handed out
  // in CTA-step chunks to whichever CTA of the group asks first (balances SMs that stream at
  // different rates: measured 34-41 us per static 1/148 of configs[1])
  const bool pool = p.pool_chunks > 0;
  const int per = pool ? p.static_keys : (n_k + p.splits - 1) / p.splits;
  const int k_lo = split * per, k_hi = min(n_k, k_lo + per);
  const size_t row_stride = (size_t)p.H * D;  // elements between consecutive keys
  const __nv_bfloat16* kb = static_cast<const __nv_bfloat16*>(p.k) + ((size_t)b * n_k * p.H + h0 + hl) * D + cidx * 8;
  const __nv_bfloat16* vb = static_cast<const __nv_bfloat16*>(p.v) + ((size_t)b * n_k * p.H + h0 + hl) * D + cidx * 8;
  const int bh = b * p.H + h0 + hl;
  SQ_T(0)

  float qf[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.q) + (size_t)bh * D + cidx * 8), qf);
#pragma unroll
  for (int i = 0; i < 8; ++i) qf[i] *= p.c;

  State st;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) st.a[i] = 0.f;

  // Per-group stream update over 4 keys x kUnroll steps per iteration (one rescale per 4 keys),
  // the CTA streaming its static key range [k_lo, k_hi). (Measured and rejected: warps claiming
  // 16 KiB chunks from a per-group counter to balance SMs that stream at different rates — the
  // claims' latency under load made it 1.3-1.45x slower at 2^22-2^24 keys and for the decode batch.)
  constexpr int KW = KS;                             // key slots per CTA
  constexpr int kWStep = 4 * KW;                     // keys per step
  const int kslot = ks;
  auto run_keys = [&](int lo, int hi, int base_first) {
    // the trip count must be warp-uniform (the shuffles below take the full mask)
    for (int base0 = lo; base0 + base_first < hi; base0 += kWStep * kUnroll) {
      const int base = base0 + kslot;
      uint4 kr[kUnroll][4], vr[kUnroll][4];
#pragma unroll
      for (int s = 0; s < kUnroll; ++s)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int key = base + s * kWStep + u * KW;
          if (key < hi) {
            kr[s][u] = ld_stream<kL2Hint>(kb + (size_t)key * row_stride);
            vr[s][u] = ld_stream<kL2Hint>(vb + (size_t)key * row_stride);
          } else {
            kr[s][u] = make_uint4(0, 0, 0, 0);
            vr[s][u] = make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
      for (int s = 0; s < kUnroll; ++s) {
        float sc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float kf[8];
          bf16x8_to_f32(kr[s][u], kf);
          float dot = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) dot = fmaf(qf[i], kf[i], dot);
#pragma unroll
          for (int o = 1; o < LPR; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          const int key = base + s * kWStep + u * KW;
          sc[u] = key < hi ? dot : -INFINITY;
        }
        const float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
        const float m_new = fmaxf(st.m, mx);
        if (m_new == -INFINITY) continue;  // nothing valid yet for this group
        const float alpha = ex2_approx(st.m - m_new);
        st.l *= alpha;
#pragma unroll
        for (int i = 0; i < 8; ++i) st.a[i] *= alpha;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float pu = ex2_approx(sc[u] - m_new);
          st.l += pu;
          float vf[8];
          bf16x8_to_f32(vr[s][u], vf);
#pragma unroll
          for (int i = 0; i < 8; ++i) st.a[i] = fmaf(pu, vf[i], st.a[i]);
        }
        st.m = m_new;
      }
    }
  };
  // Pool claims: thread 0 takes chunks two ahead of use (the atomics' latency hides under a
  // chunk of streaming) and publishes chunk i in a ring slot tagged with i; every warp walks the
  // ring on its own (no CTA barrier between chunks).
  constexpr int kRing = 32;
  __shared__ unsigned long long s_ring[kRing];
  unsigned long long* const claims = p.claims + group;
  unsigned long long a0 = 0, a1 = 0;
  if (pool) {
    for (int t = threadIdx.x; t < kRing; t += kSqThreads) s_ring[t] = ~0ull;
    __syncthreads();
    if (threadIdx.x == 0) {
      a0 = atomicAdd(claims, 1ull);
      a1 = atomicAdd(claims, 1ull);
    }
  }
  const int base_first = (warp * G) / HC;
  run_keys(k_lo, k_hi, base_first);
  if (pool) {
    auto publish = [&](int i, unsigned long long raw) {
      const unsigned c = counter_finish(claims, raw);
      const unsigned long long v = ((unsigned long long)i << 32) | (c < (unsigned)p.pool_chunks ? c : 0xFFFFFFFFu);
      *reinterpret_cast<volatile unsigned long long*>(&s_ring[i % kRing]) = v;
    };
    if (threadIdx.x == 0) {
      publish(0, a0);
      publish(1, a1);
    }
    for (int i = 0;; ++i) {
      unsigned long long v;
      do {
        v = *reinterpret_cast<volatile unsigned long long*>(&s_ring[i % kRing]);
      } while (v == ~0ull || (int)(v >> 32) < i);
      if ((int)(v >> 32) != i) __trap();  // the ring lapped a warp (cannot happen at kRing >> 2)
      const unsigned c = (unsigned)v;
      if (c == 0xFFFFFFFFu) break;       // pool exhausted (later slots are never read)
      unsigned long long an = 0;
      if (threadIdx.x == 0) an = atomicAdd(claims, 1ull);
      const int lo = p.pool_begin + (int)c * p.chunk_keys;
      run_keys(lo, min(n_k, lo + p.chunk_keys), base_first);
      if (threadIdx.x == 0) publish(i + 2, an);
    }
  }
  // merge the groups of the warp that share a head (group ids equal mod HC)
#pragma unroll
  for (int gx = HC; gx < G; gx <<= 1) {
    const int off = gx * LPR;
    State o;
    o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
    o.l = __shfl_xor_sync(0xffffffffu, st.l, off);
#pragma unroll
    for (int i = 0; i < 8; ++i) o.a[i] = __shfl_xor_sync(0xffffffffu, st.a[i], off);
    merge_state(st, o);
  }
  SQ_T(1)
  // groups g < min(G, HC) of each warp now hold distinct (warp, head) states
  constexpr int GV = G < HC ? G : HC;
  __shared__ float sm_m[NG], sm_l[NG];
  __shared__ __align__(16) float sm_a[NG][D];
  if (g < GV) {
    if (cidx == 0) {
      sm_m[gid] = st.m;
      sm_l[gid] = st.l;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sm_a[gid][cidx * 8 + i] = st.a[i];
  }
  __syncthreads();
  // CTA record per head: fold the NE states of head hl2 (entries hl2 + j * ESTEP) against their
  // common max, all loads independent (the fold is on every CTA's tail)
  constexpr int NE = HC <= G ? kSqWarps : KS;
  constexpr int ESTEP = HC <= G ? G : HC;
  for (int t = threadIdx.x; t < HC * D; t += kSqThreads) {
    const int hl2 = t / D, f = t % D;
    float mj[NE];
    float M = -INFINITY;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      mj[j] = sm_m[hl2 + j * ESTEP];
      M = fmaxf(M, mj[j]);
    }
    float l = 0.f, a = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const float w = ex2_approx(mj[j] - M);
        l = fmaf(w, sm_l[hl2 + j * ESTEP], l);
        a = fmaf(w, sm_a[hl2 + j * ESTEP][f], a);
      }
    }
    float* dst = p.rec + ((size_t)(b * p.H + h0 + hl2) * p.splits + split) * (D + 2);
    if (f == 0) {
      dst[0] = M;
      dst[1] = l;
    }
    dst[2 + f] = a;
  }
  // the final merge reuses the state arrays as scratch: (3 T O floats, T O <= max(512, HC D))
  static_assert(3 * (kSqThreads > HC * D ? kSqThreads : HC * D) <= NG * D, "merge scratch");
  __syncthreads();
  SQ_T(2)
  finish_cta<kSqThreads>(p, group, b * p.H + h0, HC, D, &sm_a[0][0]);
}

// f32 inputs, any d <= 128: one warp per key, lanes own dims {lane, lane+32, lane+64, lane+96}.
constexpr int kF32Threads = 128;
__global__ void __launch_bounds__(kF32Threads) sq_f32_kernel(const SqParams p) {
  const int split = blockIdx.x, bh = blockIdx.y;
  const int H = p.H, d = p.d, n_k = p.n_k;
  const int b = bh / H, h = bh % H;
  const float* q = static_cast<const float*>(p.q);
  const float* k = static_cast<const float*>(p.k);
  const float* v = static_cast<const float*>(p.v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (n_k + p.splits - 1) / p.splits;
  const int k_lo = split * per, k_hi = min(n_k, k_lo + per);
  float qf[4], a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) qf[i] = (lane + 32 * i < d) ? q[(size_t)bh * d + lane + 32 * i] : 0.f;
  float m = -INFINITY, l = 0.f;
  for (int key = k_lo + warp; key < k_hi; key += 4) {
    const size_t off = (((size_t)b * n_k + key) * H + h) * d;
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < d) dot = fmaf(qf[i], k[off + lane + 32 * i], dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float s = dot * p.c;
    const float m_new = fmaxf(m, s);
    const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
    const float pr = exp2f(s - m_new);
    l = l * alpha + pr;
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = a[i] * alpha + ((lane + 32 * i < d) ? pr * v[off + lane + 32 * i] : 0.f);
    m = m_new;
  }
  __shared__ float sm_m[4], sm_l[4];
  __shared__ __align__(16) float sm_a[4 * 128];   // warp states, then the merge scratch (3 x 128)
  if (lane == 0) {
    sm_m[warp] = m;
    sm_l[warp] = l;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) sm_a[warp * 128 + lane + 32 * i] = a[i];
  __syncthreads();
  if (threadIdx.x < d) {
    const int f = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w]);
    float ls = 0.f, as = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < 4; ++w) {
        const float wt = exp2f(sm_m[w] - M);
        ls += wt * sm_l[w];
        as += wt * sm_a[w * 128 + f];
      }
    float* dst = p.rec + ((size_t)bh * p.splits + split) * (d + 2);
    if (f == 0) {
      dst[0] = M;
      dst[1] = ls;
    }
    dst[2 + f] = as;
  }
  __syncthreads();
  finish_cta<kF32Threads>(p, bh, bh, 1, d, sm_a);
}

// Cross-rank merge: P triples with natural-log m. One warp per row (a (b,h)
// of a single query, or a (b, query, h) row of self-attention), lanes over the d features.
// Triple i of row r: m at m[(i*rows + r) * ms], s at s[...], v* at vstar[(i*rows + r) * vs + f]
// (separate arrays: ms = 1, vs = d; packed records {v*[d], m, s, pad, pad}: ms = vs = d + 4).
__global__ void merge_partials_kernel(const float* __restrict__ m, const float* __restrict__ s,
                                      const float* __restrict__ vstar, int64_t ms, int64_t vs, int P, int64_t rows,
                                      int d, void* out, int out_f32) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float M = -INFINITY;
  for (int i = 0; i < P; ++i) M = fmaxf(M, m[((size_t)i * rows + r) * ms]);
  float L = 0.f, A[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < P; ++i) {
    const float mi = m[((size_t)i * rows + r) * ms];
    const float w = (mi == -INFINITY) ? 0.f : expf(mi - M);
    L += w * s[((size_t)i * rows + r) * ms];
    const float* vi = vstar + ((size_t)i * rows + r) * vs;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (lane + 32 * j < d) A[j] += w * vi[lane + 32 * j];
  }
  const float inv = 1.f / L;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int f = lane + 32 * j;
    if (f >= d) break;
    if (out_f32) static_cast<float*>(out)[(size_t)r * d + f] = A[j] * inv;
    else static_cast<__nv_bfloat16*>(out)[(size_t)r * d + f] = __float2bfloat16_rn(A[j] * inv);
  }
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}



}  // namespace

// Plan: heads per CTA (HC) and key splits. HC = the largest power of two <= 4 dividing H (a
// CTA then streams HC adjacent rows per key); splits so that the grid fills the SMs (one
// 512-thread CTA per SM keeps ~128 KB of loads in flight, HBM needs ~50 KB per SM), with at
// least ~1024 keys per split.
SqPlan sq_plan(int64_t B, int64_t H, int64_t n_k, int64_t d, int bf16) {
  SqPlan pl{};
  int hc = 1;
  if (bf16) {
    // 4 adjacent head rows per key (512 B contiguous at d = 64) measured best for a decode batch
    // (16 heads x 2^20 keys: 7.0-7.2 TB/s vs 6.9 at 8 or 16 and 4.0-4.5 head-strided); the
    // merge scratch bounds HC * d (sq_bf16_kernel)
    const int lim = d == 128 ? 8 : 16;
    const int cap = g_sq_heads_per_cta > 0 ? (g_sq_heads_per_cta < lim ? g_sq_heads_per_cta : lim) : 4;
    while (hc * 2 <= cap && H % (hc * 2) == 0) hc *= 2;
  }
  pl.hc = hc;
  const int64_t groups = B * H / hc;
  const int64_t per_sm = g_sq_ctas_per_sm > 0 ? g_sq_ctas_per_sm : 1;
  const int64_t target = (bf16 ? per_sm * num_sms() : 4 * num_sms());
  // one wave: the largest split count whose grid fits the SMs, when that still fills >= 85 % of
  // them; otherwise (e.g. 100 groups on 148 SMs) more splits than fit, balanced by the pool below
  int64_t splits = target / groups;
  bool overfull = false;
  if (splits < 1 || groups * splits < target * 85 / 100) {
    splits = (target + groups - 1) / groups;
    overfull = groups * splits > target;
  }
  const int64_t max_by_keys = (n_k + 1023) / 1024;
  if (splits > max_by_keys) splits = max_by_keys;
  if (splits < 1) splits = 1;
  if (splits > 4096) splits = 4096;
  pl.splits = (int)splits;
  pl.groups = groups;
  // dynamic pool (bf16): chunks of one CTA step (4 keys x kUnroll per key slot, NG / hc slots);
  // each split keeps g_sq_static_pct % of its share as a static range; only when every split
  // still has >= 2 static chunks and the pool has >= 1 chunk per split
  pl.static_keys = 0;
  pl.chunk_keys = 0;
  pl.pool_begin = 0;
  pl.pool_chunks = 0;
  // static share: the knob, else 100 % for a single wave (a pool measured no faster there:
  // the SMs share one HBM, a fast SM does not steal bandwidth from a slow one) and 0 % when the
  // grid overfills the SMs (late CTAs find the pool drained instead of adding a second wave)
  const int pct = g_sq_static_pct >= 0 ? g_sq_static_pct : (overfull ? 0 : 100);
  if (bf16 && pct < 100) {
    const int64_t ng = (int64_t)kSqWarps * (32 / (d / 8));
    const int64_t chunk = 4 * (ng / hc) * kUnroll;
    const int64_t total = (n_k + chunk - 1) / chunk;
    const int64_t sc = total * pct / 100 / splits;
    const int64_t pool = total - sc * splits;
    if ((sc >= 2 || pct == 0) && pool >= splits) {
      pl.chunk_keys = (int)chunk;
      pl.static_keys = (int)(sc * chunk);
      pl.pool_begin = (int)(sc * chunk * splits);
      pl.pool_chunks = (int)((n_k - pl.pool_begin + chunk - 1) / chunk);
    }
  }
  pl.rec_bytes = ((size_t)B * H * splits * (d + 2) * sizeof(float) + 255) & ~(size_t)255;
  pl.bytes = pl.rec_bytes + 2 * (size_t)groups * sizeof(unsigned long long);   // tickets, claims
  return pl;
}

cudaError_t launch_sq(SqParams p, const SqPlan& pl, int bf16, cudaStream_t s) {
  p.splits = pl.splits;
  p.tickets = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(p.rec) + pl.rec_bytes);
  p.claims = pl.pool_chunks > 0 ? p.tickets + pl.groups : nullptr;
  p.static_keys = pl.static_keys;
  p.chunk_keys = pl.chunk_keys;
  p.pool_begin = pl.pool_begin;
  p.pool_chunks = pl.pool_chunks;
  if (!bf16) {
    sq_f32_kernel<<<dim3(pl.splits, (unsigned)(p.B * p.H)), kF32Threads, 0, s>>>(p);
    return cudaGetLastError();
  }
  const dim3 grid(pl.splits, (unsigned)pl.groups);
#define MEA_SQ_LAUNCH(D, HC)                                                         \
  do {                                                                               \
    if (g_sq_l2_256) sq_bf16_kernel<D, HC, true><<<grid, kSqThreads, 0, s>>>(p);     \
    else sq_bf16_kernel<D, HC, false><<<grid, kSqThreads, 0, s>>>(p);                \
  } while (0)
  if (p.d == 64) {
    switch (pl.hc) {
      case 1: MEA_SQ_LAUNCH(64, 1); break;
      case 2: MEA_SQ_LAUNCH(64, 2); break;
      case 4: MEA_SQ_LAUNCH(64, 4); break;
      case 8: MEA_SQ_LAUNCH(64, 8); break;
      default: MEA_SQ_LAUNCH(64, 16); break;
    }
  } else {
    switch (pl.hc) {
      case 1: MEA_SQ_LAUNCH(128, 1); break;
      case 2: MEA_SQ_LAUNCH(128, 2); break;
      case 4: MEA_SQ_LAUNCH(128, 4); break;
      default: MEA_SQ_LAUNCH(128, 8); break;
    }
  }
#undef MEA_SQ_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_merge_partials(const float* m, const float* s, const float* vstar, int64_t ms, int64_t vs, int P,
                                  int64_t rows, int d, void* out, int out_f32, cudaStream_t st) {
  merge_partials_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(m, s, vstar, ms, vs, P, rows, d, out, out_f32);
  return cudaGetLastError();
}

#ifdef MEA_SQ_TIMING
extern "C" __attribute__((visibility("default"))) int mea_debug_sq_times(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_sq_times, sizeof(unsigned long long) * 8 * (n < 8192 ? n : 8192));
}
#endif

}  // namespace mea
