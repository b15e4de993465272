// Streamed multi-RHS Schur reduction for sm_100a.
//
// Replaces the tile loop of reduce_group (proj/core/src/kkt.cpp:385-462):
// per scenario i and column tile V = [e_j0 .. e_j0+K)
//   X = G_x^{-1} G_u V            (T = -X)        kkt.cpp:388-404
//   acc += K_xu' T                                 kkt.cpp:430-447
//   S = K~_xx T + K_xu V                           kkt.cpp:406-423
//   Y = G_x^{-T} S ;  acc -= G_u' Y                kkt.cpp:427-447
// and acc summed over the CTA's scenarios is one column tile of the partial
// K_hat (the K_uu V term is summed by kuu_sum_kernel).
//
// Warp specialisation: warp 16 is a producer that walks the static step
// program (host/stream_plan.cpp) and stages each step's pattern block and
// values into a shared-memory ring with cp.async.bulk (TMA) on an mbarrier
// (full[]), waiting on empty[] before it overwrites a region; warps 0-15
// consume the steps on the n_x x K panel X held in shared memory, one named
// barrier per step.  Nothing on the consumers' critical path touches global
// memory except the per-scenario scatter and the S round trip.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "reduce_stream.hpp"
#include "../host/stream_plan.hpp"
#include "stats.hpp"

namespace bipm {

namespace {

constexpr int kNB = 32;  // mbarrier slots (> producer lookahead)
constexpr int kMaxQ = kStreamMaxQ;

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

enum : int { kScatter = 0, kSweep = 1, kDense = 2, kAcc = 3, kSpmv = 4, kCopyBack = 5,
             kDenseG = 6, kSweepW = 7, kScatterY = 8, kAccTail = 9,
             kStoreTail = 10 };
constexpr int kStepHeaderIntsDev = 16;  // host/stream_plan.hpp kStepHeaderInts
constexpr int kArrDenseDev = 1;         // host/stream_plan.hpp kArrDense

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
template <int C>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(C) : "memory");
}

// ring word of a step (engine.cu: ring_word): byte offset in the ring (bits
// 0-17), the barrier flags of an accumulation step (bit 18 after, bit 19
// before), and its last control (bits 20-31; 4095: never skipped)
constexpr unsigned kRwOffMask = 0x3ffffu, kRwPost = 1u << 18, kRwPre = 1u << 19;
__device__ __forceinline__ bool acc_skipped(unsigned rw, int j0) {
  const int hi = int(rw >> 20);
  return hi != 4095 && hi < j0;
}

// ---------------------------------------------------------------- panel
// Row r of the K-column panel is K*8 bytes of 16-byte chunks, chunk c at
// position c ^ sw(r) (host/stream_plan.hpp panel_word); rows are addressed by
// their precomputed word w(r) = r*K*8 + 16*sw(r) and chunk c of row r lives
// at byte w(r) ^ (c << 4).  A work unit covers CW = min(K, 8) columns.
__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds1(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void sts1(unsigned a, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ int ldsi(unsigned a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 ldsi4(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

template <int K>
struct Panel {
  static constexpr int CW = K < kStreamUnitCols ? K : kStreamUnitCols;  // columns per unit
  static constexpr int NG = K / CW;         // unit groups per row
  static constexpr int NC = CW / 2;         // 16-byte chunks per unit
  __host__ __device__ static constexpr int swz(int r) {
    return K >= 16 ? (r & 7) : K == 8 ? ((r >> 1) & 3) : K == 4 ? ((r >> 2) & 1) : 0;
  }
  __device__ static int word(int r) { return r * K * 8 + 16 * swz(r); }
  // a += v * X[row w, columns of group cg]
  __device__ static void fma(double (&a)[CW], double v, unsigned xb, int w, int cg) {
    if constexpr (K == 1) {
      a[0] += v * lds1(xb + w);
    } else {
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const double2 x = lds2(xb + (w ^ ((cg * NC + q) << 4)));
        a[2 * q] += v * x.x;
        a[2 * q + 1] += v * x.y;
      }
    }
  }
  __device__ static void load(double (&x)[CW], unsigned xb, int w, int cg) {
    if constexpr (K == 1) {
      x[0] = lds1(xb + w);
    } else {
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const double2 t = lds2(xb + (w ^ ((cg * NC + q) << 4)));
        x[2 * q] = t.x;
        x[2 * q + 1] = t.y;
      }
    }
  }
  __device__ static void store(const double (&x)[CW], unsigned xb, int w, int cg) {
    if constexpr (K == 1) {
      sts1(xb + w, x[0]);
    } else {
#pragma unroll
      for (int q = 0; q < NC; ++q) sts2(xb + (w ^ ((cg * NC + q) << 4)), x[2 * q], x[2 * q + 1]);
    }
  }
  // byte offset of element (row r, column c)
  __device__ static int elem(int r, int c) {
    if constexpr (K == 1) return r * 8;
    return (word(r) ^ ((c >> 1) << 4)) + ((c & 1) << 3);
  }
};

template <int CW>
__device__ __forceinline__ void reduce_lanes(double (&a)[CW], int g) {
  for (int off = g >> 1; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < CW; ++q) a[q] += __shfl_xor_sync(0xffffffffu, a[q], off);
  }
}

__device__ __forceinline__ void acc_add(double (&acc)[kMaxQ], int q, double v) {
#pragma unroll
  for (int r = 0; r < kMaxQ; ++r)
    if (r == q) acc[r] += v;
}

// column entry t of a step -> its panel word: the entry holds word / 16
// (K >= 2) or the panel row (K = 1, word 8 r) (host/stream_plan.cpp emit)
template <int K>
__device__ __forceinline__ int colw(unsigned col, int t) {
  unsigned short r;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(col + 2 * t));
  return K == 1 ? int(r) << 3 : int(r) << 4;
}

// Step header (host/stream_plan.hpp): 16 ints
struct Hdr {
  int kind, flags, n_items, n_col, aux0, aux1, vcount, par, lg, n_units, warp0, n_lev;
};
enum : int { kFDiag = 1, kFCommit = 2, kFBarrier = 4, kFPre = 8 };

// Work-unit loop shared by the sweep / dense / spmv steps: chunks of 32 >> lg
// units (2^lg lanes each) are dealt to the warps round robin from warp0; the
// loop bound is warp-uniform so the lane reductions see full warps.
#define UNIT_LOOP(h, tid, ...)                                                   \
  {                                                                               \
    const int lg_ = (h).lg, g_ = 1 << lg_;                                       \
    const int lane_ = (tid) & 31, warp_ = (tid) >> 5;                            \
    const int upw_ = 32 >> lg_;                                                   \
    const int nch_ = ((h).n_units + upw_ - 1) >> (5 - lg_);                      \
    for (int c_ = (warp_ - (h).warp0 + C / 32) & (C / 32 - 1); c_ < nch_;      \
         c_ += C / 32) {                                                         \
      const int unit = c_ * upw_ + (lane_ >> lg_);                                \
      const int sub = lane_ & (g_ - 1);                                           \
      const bool active = unit < (h).n_units;                                     \
      const int g = g_;                                                           \
      __VA_ARGS__                                                                 \
    }                                                                             \
  }

// one level (or part of one) of a triangular sweep: x_r -= sum v x_col, then
// divided by the diagonal (the item's first entry) with kFlagDiag
// barrier of the team of the lowest T consumer warps (T = C/32: all of them,
// barrier 1; T = 1: the warp itself)
template <int C>
__device__ __forceinline__ void team_sync(int T) {
  if (T == C / 32) {
    consumer_sync<C>();
    return;
  }
  switch (T) {
    case 8: asm volatile("bar.sync 2, 256;" ::: "memory"); break;
    case 4: asm volatile("bar.sync 3, 128;" ::: "memory"); break;
    case 2: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
    default: __syncwarp(); break;
  }
}

// debug trace (CTA (0,0), thread 0, first scenario): (code, clock64) pairs,
// compiled in with -DBIPM_TRACE (tools/trace_reduce.py)
struct Tracer {
  long long* buf = nullptr;
  int n = 0;
  __device__ void operator()(int code) {
#ifdef BIPM_TRACE
    if (buf && n < 30000) {
      buf[2 * n] = code;
      buf[2 * n + 1] = clock64();
      ++n;
    }
#else
    (void)code;
#endif
  }
};

template <int K, int C>
__device__ __forceinline__ void step_sweep(const Hdr& h, unsigned lev, unsigned items,
                                           unsigned col, unsigned v, unsigned xb, int tid,
                                           Tracer& tr, int dbg) {
  using Pn = Panel<K>;
  const int T = h.aux0, warp = tid >> 5, lane = tid & 31;
  if (warp >= T) return;
  if (dbg & 1) return;
  const int dg = h.flags & 1;
  for (int L = 0; L < h.n_lev; ++L) {
    const int4 e = ldsi4(lev + 16 * L);  // unit begin, unit end, lg, barrier
    const int lg = e.z, g = 1 << lg, upw = 32 >> lg;
    const int nch = (e.y - e.x + upw - 1) >> (5 - lg);
    const int sub = lane & (g - 1);
    tr(100 + L);
    for (int c = warp; c < nch; c += T) {
      const int unit = e.x + c * upw + (lane >> lg);
      const bool active = unit < e.y;
      const int item = Pn::NG == 1 ? unit : unit / Pn::NG;
      const int cg = Pn::NG == 1 ? 0 : unit % Pn::NG;
      double a[Pn::CW];
#pragma unroll
      for (int q = 0; q < Pn::CW; ++q) a[q] = 0.0;
      int4 m = make_int4(0, 0, 0, 0);
      if (active) {
        m = ldsi4(items + 16 * item);
        int t = m.y + dg + sub;
        // K = 1 (one 8-byte gather per entry): four entries' loads in flight
        // (9241/16: -4 %); wider panels measured slower with it (+2-3 %)
        for (; K == 1 && t + 3 * g < m.z; t += 4 * g) {
          const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
          const int w2 = colw<K>(col, t + 2 * g), w3 = colw<K>(col, t + 3 * g);
          const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
          const double v2 = lds1(v + 8 * (t + 2 * g)), v3 = lds1(v + 8 * (t + 3 * g));
          Pn::fma(a, v0, xb, w0, cg);
          Pn::fma(a, v1, xb, w1, cg);
          Pn::fma(a, v2, xb, w2, cg);
          Pn::fma(a, v3, xb, w3, cg);
        }
        for (; t + g < m.z; t += 2 * g) {
          const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
          const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
          Pn::fma(a, v0, xb, w0, cg);
          Pn::fma(a, v1, xb, w1, cg);
        }
        if (t < m.z) Pn::fma(a, lds1(v + 8 * t), xb, colw<K>(col, t), cg);
      }
      reduce_lanes<Pn::CW>(a, g);
      if (active && sub == 0) {
        double x[Pn::CW];
        Pn::load(x, xb, m.x, cg);
        if (dg) {
          const double r = 1.0 / lds1(v + 8 * m.y);
#pragma unroll
          for (int q = 0; q < Pn::CW; ++q) x[q] = (x[q] - a[q]) * r;
        } else {
#pragma unroll
          for (int q = 0; q < Pn::CW; ++q) x[q] -= a[q];
        }
        Pn::store(x, xb, m.x, cg);
      }
    }
    tr(200 + L);
    if (e.w && !(dbg & 2)) team_sync<C>(T);
    tr(300 + L);
  }
}

// warp-local part of a triangular sweep (host/stream_plan.cpp, subtree
// mapping): warp w runs its own levels [dir[w].x, dir[w].y) -- rows of the
// elimination subtrees assigned to it -- separated by __syncwarp only.  The
// subtrees are disjoint and closed under the sweep's dependencies, so no
// other warp reads or writes these rows until the next all-consumer barrier.
template <int K, int C>
__device__ __forceinline__ void step_sweep_w(const Hdr& h, unsigned dir, unsigned lev,
                                             unsigned items, unsigned col, unsigned v,
                                             unsigned xb, int tid) {
  using Pn = Panel<K>;
  const int warp = tid >> 5, lane = tid & 31;
  const int dg = h.flags & 1;
  const int2 d = make_int2(ldsi(dir + 8 * warp), ldsi(dir + 8 * warp + 4));
  for (int L = d.x; L < d.y; ++L) {
    const int4 e = ldsi4(lev + 16 * L);  // unit begin, unit end, lg
    const int lg = e.z, g = 1 << lg, upw = 32 >> lg;
    const int nch = (e.y - e.x + upw - 1) >> (5 - lg);
    const int sub = lane & (g - 1);
    for (int c = 0; c < nch; ++c) {
      const int unit = e.x + c * upw + (lane >> lg);
      const bool active = unit < e.y;
      const int item = Pn::NG == 1 ? unit : unit / Pn::NG;
      const int cg = Pn::NG == 1 ? 0 : unit % Pn::NG;
      double a[Pn::CW];
#pragma unroll
      for (int q = 0; q < Pn::CW; ++q) a[q] = 0.0;
      int4 m = make_int4(0, 0, 0, 0);
      if (active) {
        m = ldsi4(items + 16 * item);
        int t = m.y + dg + sub;
        // K = 1 (one 8-byte gather per entry): four entries' loads in flight
        // (9241/16: -4 %); wider panels measured slower with it (+2-3 %)
        for (; K == 1 && t + 3 * g < m.z; t += 4 * g) {
          const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
          const int w2 = colw<K>(col, t + 2 * g), w3 = colw<K>(col, t + 3 * g);
          const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
          const double v2 = lds1(v + 8 * (t + 2 * g)), v3 = lds1(v + 8 * (t + 3 * g));
          Pn::fma(a, v0, xb, w0, cg);
          Pn::fma(a, v1, xb, w1, cg);
          Pn::fma(a, v2, xb, w2, cg);
          Pn::fma(a, v3, xb, w3, cg);
        }
        for (; t + g < m.z; t += 2 * g) {
          const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
          const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
          Pn::fma(a, v0, xb, w0, cg);
          Pn::fma(a, v1, xb, w1, cg);
        }
        if (t < m.z) Pn::fma(a, lds1(v + 8 * t), xb, colw<K>(col, t), cg);
      }
      reduce_lanes<Pn::CW>(a, g);
      if (active && sub == 0) {
        double x[Pn::CW];
        Pn::load(x, xb, m.x, cg);
        if (dg) {
          const double r = 1.0 / lds1(v + 8 * m.y);
#pragma unroll
          for (int q = 0; q < Pn::CW; ++q) x[q] = (x[q] - a[q]) * r;
        } else {
#pragma unroll
          for (int q = 0; q < Pn::CW; ++q) x[q] -= a[q];
        }
        Pn::store(x, xb, m.x, cg);
      }
    }
    __syncwarp();
  }
}

// rows [r0, r0 + nr) of X_T <- W X_T (W row-major tl x tl in the ring) into
// temp (row-major, K per row)
template <int K, int C>
__device__ __forceinline__ void step_dense(const Hdr& h, unsigned W, unsigned xb, double* temp,
                                           int t0, int tl, int tid) {
  using Pn = Panel<K>;
  const int r0 = h.aux0;
  UNIT_LOOP(h, tid, {
    const int i = Pn::NG == 1 ? unit : unit / Pn::NG;
    const int cg = Pn::NG == 1 ? 0 : unit % Pn::NG;
    double a[Pn::CW];
_Pragma("unroll")
    for (int q = 0; q < Pn::CW; ++q) a[q] = 0.0;
    if (active) {
      const unsigned wr = W + 8 * i * tl;
      int k = sub;
      for (; k + g < tl; k += 2 * g) {
        const double w0 = lds1(wr + 8 * k), w1 = lds1(wr + 8 * (k + g));
        Pn::fma(a, w0, xb, Pn::word(t0 + k), cg);
        Pn::fma(a, w1, xb, Pn::word(t0 + k + g), cg);
      }
      if (k < tl) Pn::fma(a, lds1(wr + 8 * k), xb, Pn::word(t0 + k), cg);
    }
    reduce_lanes<Pn::CW>(a, g);
    if (active && sub == 0) {
_Pragma("unroll")
      for (int q = 0; q < Pn::CW; ++q) temp[(r0 + i) * K + cg * Pn::CW + q] = a[q];
    }
  })
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// temp = W X_T for the whole tail on the FP64 tensor pipe (DMMA m8n8k4):
// warp = 8 output rows x all K columns; A = W rows from global memory (L2,
// eight k-steps of loads in flight), B = X_T from the panel in shared memory
// (general form: temp[i K + c] = sum_k A(i, k) X[t0 + k, c] for i < m, k < tl,
// A rows k-contiguous with stride lda (a multiple of 16 doubles))
template <int K, int C>
__device__ __forceinline__ void step_dense_global(const double* __restrict__ W, unsigned xb,
                                                  double* temp, int t0, int tl, int tid,
                                                  int m = -1, int lda = -1) {
  using Pn = Panel<K>;
  constexpr int NT = K >= 8 ? K / 8 : 1;  // 8-column tiles
  const int lane = tid & 31, warp = tid >> 5;
  const int gm = lane >> 2, gk = lane & 3;
  if (m < 0) m = tl;
  const int ldw = lda >= 0 ? lda : (tl + 15) & ~15;  // host/stream_plan.hpp dense_ld
  const int mtiles = (m + 7) >> 3;
  for (int mt = warp; mt < mtiles; mt += C / 32) {
    const int i = mt * 8 + gm;
    // lane (gm, gk) reads W(i, k0 + 4 gk .. +3) as one 32-byte vector: the 4
    // lanes of a row cover one 128-byte line, and DMMA step j of the chunk
    // takes k = k0 + 4 gk + j (any k order works when A and B agree)
    const double* __restrict__ wr = W + size_t(i < m ? i : 0) * ldw + 4 * gk;
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
    auto ld = [&](int k0, double (&r)[4]) {
      if (k0 < tl) {
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                     : "l"(wr + k0));
      } else {
        r[0] = r[1] = r[2] = r[3] = 0.0;
      }
    };
    auto chunk = [&](int k0, const double (&r)[4]) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + 4 * gk + j;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int c = n * 8 + gm;
          const double bf = (k < tl && c < K) ? lds1(xb + Pn::elem(t0 + k, c)) : 0.0;
          dmma884(acc[n][0], acc[n][1], r[j], bf);
        }
      }
    };
    // three 16-column chunks in flight (W comes from L2)
    double r0[4], r1[4], r2[4];
    ld(0, r0);
    ld(16, r1);
    ld(32, r2);
    for (int k0 = 0; k0 < tl; k0 += 48) {
      chunk(k0, r0);
      ld(k0 + 48, r0);
      if (k0 + 16 >= tl) break;
      chunk(k0 + 16, r1);
      ld(k0 + 64, r1);
      if (k0 + 32 >= tl) break;
      chunk(k0 + 32, r2);
      ld(k0 + 80, r2);
    }
    if (i < m) {
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int c = n * 8 + 2 * gk + v;
          if (c < K) temp[i * K + c] = acc[n][v];
        }
    }
  }
}

// S_p = -(sum_t kxx_t X_col + (sigma_x,i + dw) X_p) over a range of state rows;
// S (global scratch) uses the panel layout
template <int K, int C>
__device__ __forceinline__ void step_spmv(const Hdr& h, unsigned items, unsigned col, unsigned v,
                                          unsigned sig, unsigned xb, char* S, double dw,
                                          int tid, int dbg = 0) {
  using Pn = Panel<K>;
  UNIT_LOOP(h, tid, {
    const int item = Pn::NG == 1 ? unit : unit / Pn::NG;
    const int cg = Pn::NG == 1 ? 0 : unit % Pn::NG;
    double a[Pn::CW];
_Pragma("unroll")
    for (int q = 0; q < Pn::CW; ++q) a[q] = 0.0;
    int4 m = make_int4(0, 0, 0, 0);
    if (active) {
      m = ldsi4(items + 16 * item);
      int t = m.y + sub;
      for (; K == 1 && t + 3 * g < m.z; t += 4 * g) {  // K = 1: four entries in flight
        const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
        const int w2 = colw<K>(col, t + 2 * g), w3 = colw<K>(col, t + 3 * g);
        const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
        const double v2 = lds1(v + 8 * (t + 2 * g)), v3 = lds1(v + 8 * (t + 3 * g));
        Pn::fma(a, v0, xb, w0, cg);
        Pn::fma(a, v1, xb, w1, cg);
        Pn::fma(a, v2, xb, w2, cg);
        Pn::fma(a, v3, xb, w3, cg);
      }
      for (; t + g < m.z; t += 2 * g) {
        const int w0 = colw<K>(col, t), w1 = colw<K>(col, t + g);
        const double v0 = lds1(v + 8 * t), v1 = lds1(v + 8 * (t + g));
        Pn::fma(a, v0, xb, w0, cg);
        Pn::fma(a, v1, xb, w1, cg);
      }
      if (t < m.z) Pn::fma(a, lds1(v + 8 * t), xb, colw<K>(col, t), cg);
    }
    reduce_lanes<Pn::CW>(a, g);
    if (active && sub == 0 && !(dbg & 4)) {  // dbg 4: timing experiment without the S stores
      double x[Pn::CW];
      Pn::load(x, xb, m.x, cg);
      const double d = lds1(sig + 8 * m.w) + dw;
      if constexpr (K == 1) {
        *reinterpret_cast<double*>(S + m.x) = -(a[0] + d * x[0]);
      } else {
_Pragma("unroll")
        for (int q = 0; q < Pn::NC; ++q)
          *reinterpret_cast<double2*>(S + (m.x ^ ((cg * Pn::NC + q) << 4))) =
              make_double2(-(a[2 * q] + d * x[2 * q]), -(a[2 * q + 1] + d * x[2 * q + 1]));
      }
    }
  })
}

// acc -= A' X over controls [u0, u0 + n_items) of accumulator register q; the
// consumer owning (u, c) is (u K + c) mod 512
template <int K, int C>
__device__ __forceinline__ void step_acc(const Hdr& h, unsigned items, unsigned col, unsigned v,
                                         unsigned xb, double (&acc)[kMaxQ], int tid, int j0) {
  // the step's controls [u0, u0 + n_items) may span several accumulator
  // registers q (control u of column c lives in register q = u / (C / K)).
  // Only the lower triangle of K_hat is assembled (finish_reduce mirrors it):
  // entries u < j0 + c are skipped
  const int u0 = h.aux1, n = h.n_items, c = tid % K;
  const int cx = K == 1 ? 0 : (((c >> 1) << 4));
  const int co = K == 1 ? 0 : ((c & 1) << 3);
  for (int q = u0 / (C / K); q * (C / K) < u0 + n; ++q) {
    const int u = q * (C / K) + tid / K;
    const int it = u - u0;
    if (it >= 0 && it < n && u >= j0 + c) {
      const int4 m = ldsi4(items + 16 * it);
      double a0 = 0.0, a1 = 0.0;
      int t = m.y;
      for (; t + 1 < m.z; t += 2) {
        a0 += lds1(v + 8 * t) * lds1(xb + (colw<K>(col, t) ^ cx) + co);
        a1 += lds1(v + 8 * (t + 1)) * lds1(xb + (colw<K>(col, t + 1) ^ cx) + co);
      }
      if (t < m.z) a0 += lds1(v + 8 * t) * lds1(xb + (colw<K>(col, t) ^ cx) + co);
      acc_add(acc, q, -(a0 + a1));
    }
  }
}

template <int K, int C>
__global__ void __launch_bounds__(C + 32, 512 / C) reduce_stream_kernel(StreamLaunch a) {
  constexpr int kThreads = C + 32;
  using Pn = Panel<K>;
  extern __shared__ __align__(1024) unsigned char smem[];
  // layout: X panel (offset 0, 256-byte aligned rows) | barriers | ring
  // offsets | tile lists | ring.  The dense-tail product's output stages in
  // the CTA's global scratch S (free while the dense steps run: S carries
  // K~_xx T only from the product steps to the copy-back), which leaves its
  // tl x K doubles of shared memory to the ring.
  const int P = a.steps;
  double* X = reinterpret_cast<double*>(smem);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(X + size_t(a.n_x) * K);
  unsigned long long* empty = full + kNB;
  int* ring_off = reinterpret_cast<int*>(empty + kNB);
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int j0 = tile * K;
  const int k = min(K, a.n_u - j0);
  // tile lists: (panel byte offset, slot) of the tile's G_u and K_xu columns
  // tile lists in the CTA's global scratch, after S (n_x K doubles): read
  // once per scenario, so shared memory goes to the ring instead
  double* cta_scratch =
      a.scratch + size_t(chunk * gridDim.x + tile) * (size_t(a.n_x) * K + a.list_cap);
  int2* gu_list = reinterpret_cast<int2*>(cta_scratch + size_t(a.n_x) * K);
  // presolved: the "G_u" list holds the tile's y_N entries instead
  const int n_gu = a.presolved ? a.yn_ptr[j0 + k] - a.yn_ptr[j0]
                               : a.gu.t_ptr[j0 + k] - a.gu.t_ptr[j0];
  const int n_kxu = a.kxu.t_ptr[j0 + k] - a.kxu.t_ptr[j0];
  int2* kxu_list = gu_list + ((n_gu + 1) & ~1);
  unsigned char* ring = reinterpret_cast<unsigned char*>(ring_off + ((P + 3) & ~3));
  ring = reinterpret_cast<unsigned char*>((reinterpret_cast<size_t>(ring) + 15) & ~size_t(15));
  const unsigned xb = smem_u32(X), rb = smem_u32(ring);

  const int tid = threadIdx.x;
  const int s_lo = chunk * a.chunk, s_hi = min(a.M, s_lo + a.chunk);
  const int total = (s_hi - s_lo) * P;
  if (tid == 0) {
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], C / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < P; j += kThreads) ring_off[j] = a.ring_off[j];
  if (a.presolved) {
    for (int e = tid; e < n_gu; e += kThreads) {
      const int q = a.yn_ptr[j0] + e;
      int c = 0;
      while (a.yn_ptr[j0 + c + 1] <= q) ++c;
      gu_list[e] = make_int2(Pn::elem(a.yn_row[q], c), q);
    }
  } else {
    for (int e = tid; e < n_gu; e += kThreads) {
      const int q = a.gu.t_ptr[j0] + e;
      int c = 0;
      while (a.gu.t_ptr[j0 + c + 1] <= q) ++c;
      gu_list[e] = make_int2(Pn::elem(a.iperm[a.gu.t_row[q]], c), a.gu.t_slot[q]);
    }
  }
  for (int e = tid; e < n_kxu; e += kThreads) {
    const int q = a.kxu.t_ptr[j0] + e;
    int c = 0;
    while (a.kxu.t_ptr[j0 + c + 1] <= q) ++c;
    kxu_list[e] = make_int2(Pn::elem(a.iperm[a.kxu.t_row[q]], c), a.kxu.t_slot[q]);
  }
  __syncthreads();

  if (tid >= C) {  // ------------------------------------------- producer warp
    const int lane = tid - C;
    for (int jb = 0; jb < total; jb += 32) {
      int rec[12];
      {
        const int jl = jb + lane;
        const int* r = a.issue + size_t(jl < total ? jl % P : 0) * 12;
#pragma unroll
        for (int f = 0; f < 12; ++f) rec[f] = r[f];
      }
      const int nb = min(32, total - jb);
      for (int l = 0; l < nb; ++l) {
        int f[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) f[q] = __shfl_sync(0xffffffffu, rec[q], l);
        const int j = jb + l;
        const int s = s_lo + j / P;
        if (lane == 0) {
          const int wd = f[11];
          if (wd > 0 && j - wd >= 0) {
            const int w = j - wd;
            mbar_wait(&empty[w % kNB], (w / kNB) & 1);
          }
          // values: aligned-down 16-byte start, the consumer skips the shift
          unsigned vb = 0, xb2 = 0;
          const double *vsrc = nullptr, *xsrc = nullptr;
          if (f[5] > 0) {
            const long long e = (long long)s * a.stride[f[3]] + f[4];
            vsrc = a.arr[f[3]] + (e & ~1LL);
            vb = unsigned(((e & 1) + f[5]) * 8 + 15) & ~15u;
          }
          if (f[8] > 0) {
            const long long e = (long long)s * a.stride[f[6]] + f[7];
            xsrc = a.arr[f[6]] + (e & ~1LL);
            xb2 = unsigned(((e & 1) + f[8]) * 8 + 15) & ~15u;
          }
          unsigned long long* fb = &full[j % kNB];
          if (acc_skipped(ring_off[j % P], j0)) {
            mbar_arrive(fb);  // accumulation step below the tile's triangle: nothing to load
          } else {
            mbar_arrive_tx(fb, unsigned(f[1]) + vb + xb2);
            bulk_g2s(ring + f[2], a.pat + f[0], unsigned(f[1]), fb);
            if (vb) bulk_g2s(ring + f[9], vsrc, vb, fb);
            if (xb2) bulk_g2s(ring + f[10], xsrc, xb2, fb);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  double acc[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) acc[q] = 0.0;
  char* S = reinterpret_cast<char*>(cta_scratch);
  double* temp = reinterpret_cast<double*>(S);
  const int nxk2 = a.n_x * K / 2;  // 16-byte chunks of the panel (K >= 2)
  const bool stamp = a.phase && tile == 0 && chunk == 0 && tid == 0;
  Tracer tr;
  if (stamp) tr.buf = a.phase + 2 * P + 2;
  const int lane = tid & 31;

  int jj = 0, s = s_lo;
  for (int j = 0; j < total; ++j) {
    if (stamp && s == s_lo) a.phase[2 * jj] = clock64();
    if (s != s_lo) tr.buf = nullptr;
    tr(1);
    mbar_wait(&full[j & (kNB - 1)], (j / kNB) & 1);
    tr(2);
    if (stamp && s == s_lo) a.phase[2 * jj + 1] = clock64();
    const unsigned rw = unsigned(ring_off[jj]);
    if (acc_skipped(rw, j0)) {
      // skipped accumulation step (StreamProgram::skip): its barriers only
      if (rw & kRwPre) consumer_sync<C>();
      if (rw & kRwPost) consumer_sync<C>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[j & (kNB - 1)]);
      if (++jj == P) {
        jj = 0;
        ++s;
      }
      continue;
    }
    const unsigned base = rb + (rw & kRwOffMask);
    Hdr h;
    {
      const int4 h0 = ldsi4(base), h1 = ldsi4(base + 16), h2 = ldsi4(base + 32);
      h = Hdr{h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w, h2.x, h2.y, h2.z, h2.w};
    }
    // warp-local sweeps carry a per-warp directory (2 ints per consumer warp)
    const unsigned dir = base + 4 * kStepHeaderIntsDev;
    const unsigned lev = dir + (h.kind == kSweepW ? ((8 * (C / 32) + 15) & ~15) : 0);
    const unsigned items = lev + 16 * h.n_lev;
    const unsigned col = items + 16 * h.n_items;
    const unsigned vals = col + 2 * h.n_col;
    const int vshift = (h.par & 1) ^ ((h.par >> 1) & s & 1);
    const unsigned v = vals + 8 * vshift;
    tr(3);
    if (h.flags & kFPre) consumer_sync<C>();
    tr(4);
    switch (h.kind) {
      case kScatter: {
        if constexpr (K == 1) {
          for (int i = tid; i < a.n_x; i += C) sts1(xb + 8 * i, 0.0);
        } else {
          for (int i = tid; i < nxk2; i += C) sts2(xb + 16 * i, 0.0, 0.0);
        }
        consumer_sync<C>();
        const double* gu = a.gu_v + size_t(s) * a.gu.nnz;
        for (int e0 = tid; e0 < n_gu; e0 += 4 * C) {  // list and value loads in flight
          int2 l[4];
          double g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) l[u] = e0 + u * C < n_gu ? gu_list[e0 + u * C] : make_int2(0, 0);
#pragma unroll
          for (int u = 0; u < 4; ++u) g[u] = e0 + u * C < n_gu ? gu[l[u].y] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (e0 + u * C < n_gu) sts1(xb + l[u].x, g[u]);
        }
        break;
      }
      case kScatterY: {
        // X = 0; X[y_N rows, c] = y_N; X[tail, c] = X_T[:, j0 + c]
        if constexpr (K == 1) {
          for (int i = tid; i < a.n_x; i += C) sts1(xb + 8 * i, 0.0);
        } else {
          for (int i = tid; i < nxk2; i += C) sts2(xb + 16 * i, 0.0, 0.0);
        }
        consumer_sync<C>();
        const double* yv = a.yn_v + size_t(s) * a.nnz_yn;
        for (int e0 = tid; e0 < n_gu; e0 += 4 * C) {
          int2 l[4];
          double g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) l[u] = e0 + u * C < n_gu ? gu_list[e0 + u * C] : make_int2(0, 0);
#pragma unroll
          for (int u = 0; u < 4; ++u) g[u] = e0 + u * C < n_gu ? yv[l[u].y] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (e0 + u * C < n_gu) sts1(xb + l[u].x, g[u]);
        }
        const double* xt = a.xt + (size_t(s) * a.n_u + j0) * a.ldy;
        const int nt = a.tl * k;
        for (int e0 = tid; e0 < nt; e0 += 4 * C) {
          double g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * C;
            g[u] = e < nt ? xt[size_t(e / a.tl) * a.ldy + e % a.tl] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * C;
            if (e < nt) sts1(xb + Pn::elem(a.t0 + e % a.tl, e / a.tl), g[u]);
          }
        }
        break;
      }
      case kSweep:
        step_sweep<K, C>(h, lev, items, col, v, xb, tid, tr, a.debug);
        break;
      case kSweepW:
        step_sweep_w<K, C>(h, dir, lev, items, col, v, xb, tid);
        break;
      case kDense:
        step_dense<K, C>(h, v, xb, temp, a.t0, a.tl, tid);
        if (h.flags & 2) {
          consumer_sync<C>();
          for (int e = tid; e < a.tl * K; e += C)
            sts1(xb + Pn::elem(a.t0 + e / K, e % K), temp[e]);
        }
        break;
      case kDenseG: {
        const double* W = a.arr[kArrDenseDev] + size_t(s) * a.stride[kArrDenseDev] +
                          size_t(h.aux0) * a.tl * ((a.tl + 15) & ~15);
        step_dense_global<K, C>(W, xb, temp, a.t0, a.tl, tid);
        consumer_sync<C>();
        for (int e0 = tid; e0 < a.tl * K; e0 += 4 * C) {  // four L2 loads in flight
          double t[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) t[u] = e0 + u * C < a.tl * K ? temp[e0 + u * C] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * C;
            if (e < a.tl * K) sts1(xb + Pn::elem(a.t0 + e / K, e % K), t[u]);
          }
        }
        break;
      }
      case kAcc:
        step_acc<K, C>(h, items, col, v, xb, acc, tid, j0);
        break;
      case kStoreTail: {
        // Z_T of the tile's columns for the batch-sum GEMM (acc -= X_T' Z_T)
        double* zt = a.zt + (size_t(s) * a.n_u + j0) * a.ldy;
        const int nt = a.tl * k;
        for (int e = tid; e < nt; e += C) {
          const int c = e / a.tl, t = e - c * a.tl;
          zt[size_t(c) * a.ldy + t] = lds1(xb + Pn::elem(a.t0 + t, c));
        }
        break;
      }
      case kAccTail: {
        // acc -= X_T' Z_T: temp[u K + c] = sum_t X_T[t, u] Z[t0 + t, c] (the
        // temp index of (u, c) is the owner's tid + q C)
        step_dense_global<K, C>(a.xt + size_t(s) * a.n_u * a.ldy, xb, temp, a.t0, a.tl, tid,
                                a.n_u, a.ldy);
        consumer_sync<C>();
#pragma unroll
        for (int q = 0; q < kMaxQ; ++q) {
          const int it = tid + q * C;
          if (q < a.nq && it < a.n_u * K) acc[q] -= temp[it];
        }
        break;
      }
      case kSpmv: {
        const int xoff = h.vcount > 0 ? ((h.vcount + 1) * 8 + 15) & ~15 : 0;
        const int xshift = ((h.par >> 2) & 1) ^ ((h.par >> 3) & s & 1);
        step_spmv<K, C>(h, items, col, v, vals + xoff + 8 * xshift, xb, S, a.dw, tid, a.debug);
        break;
      }
      case kCopyBack: {
        // four loads of a thread in flight before its stores (sts* are
        // volatile asm with a memory clobber: a plain loop waits one L2
        // round trip per element)
        if constexpr (K == 1) {
          const double* Sd = reinterpret_cast<const double*>(S);
          for (int i0 = tid; i0 < a.n_x; i0 += 4 * C) {
            double t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = i0 + u * C < a.n_x ? Sd[i0 + u * C] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i0 + u * C < a.n_x) sts1(xb + 8 * (i0 + u * C), t[u]);
          }
        } else {
          const double2* S2 = reinterpret_cast<const double2*>(S);
          for (int i0 = tid; i0 < nxk2; i0 += 4 * C) {
            double2 t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              t[u] = i0 + u * C < nxk2 ? S2[i0 + u * C] : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i0 + u * C < nxk2) sts2(xb + 16 * (i0 + u * C), t[u].x, t[u].y);
          }
        }
        consumer_sync<C>();
        const double* kxu = a.kxu_v + size_t(s) * a.kxu.nnz;
        for (int e0 = tid; e0 < n_kxu; e0 += 4 * C) {
          int2 l[4];
          double g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            l[u] = e0 + u * C < n_kxu ? kxu_list[e0 + u * C] : make_int2(0, 0);
#pragma unroll
          for (int u = 0; u < 4; ++u) g[u] = e0 + u * C < n_kxu ? kxu[l[u].y] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (e0 + u * C < n_kxu) sts1(xb + l[u].x, lds1(xb + l[u].x) + g[u]);
        }
        break;
      }
      default:
        break;
    }
    tr(5);
    if (h.flags & kFBarrier) consumer_sync<C>();
    tr(6);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[j & (kNB - 1)]);
    if (++jj == P) {
      jj = 0;
      ++s;
    }
  }
  if (stamp) {
    a.phase[2 * P] = clock64();
    a.phase[2 * P + 1] = tr.n;
  }

  double* out = a.partial + size_t(chunk) * a.n_u * a.n_u;
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) {
    const int it = tid + q * C;
    if (q < a.nq && it < a.n_u * K) {
      const int u = it / K, c = it % K;
      if (c < k) out[size_t(j0 + c) * a.n_u + u] = acc[q];
    }
  }
}

// sum over scenarios (fixed order) of K_uu, scattered into the dense
// column-major n_u x n_u part: the K_uu V term of every column tile
__global__ void kuu_sum_kernel(const double* __restrict__ kuu, long long stride,
                               const int* __restrict__ row, const int* __restrict__ col, int nnz,
                               int M, int n_u, double* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int s = 0;
  for (; s + 3 < M; s += 4) {
    s0 += kuu[s * stride + q];
    s1 += kuu[(s + 1) * stride + q];
    s2 += kuu[(s + 2) * stride + q];
    s3 += kuu[(s + 3) * stride + q];
  }
  for (; s < M; ++s) s0 += kuu[s * stride + q];
  out[size_t(col[q]) * n_u + row[q]] = (s0 + s1) + (s2 + s3);
}

__global__ void gather_values_kernel(const double* __restrict__ in, long long in_stride,
                                     const int* __restrict__ slot, int n, double* out,
                                     long long out_stride, int M) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * M) return;
  const int s = int(t / n), q = int(t % n);
  out[s * out_stride + q] = in[s * in_stride + slot[q]];
}

}  // namespace

size_t stream_smem_bytes(int n_x, int K, int tl, int steps, int list_cap, int ring_bytes) {
  // panel + barriers + ring offsets + ring (the dense-tail output and the
  // tile lists live in global scratch: tl and list_cap are not needed here)
  (void)tl;
  (void)list_cap;
  return size_t(n_x) * K * 8 + 2 * kNB * 8 + size_t((steps + 3) & ~3) * 4 + 16 + ring_bytes;
}

int stream_ring_capacity(int n_x, int K, int tl, int steps, int list_cap, int ctas_per_sm) {
  // 228 KB of shared memory per SM, 1 KB of it reserved per resident CTA
  const long long per_cta = std::min(227LL * 1024, 228LL * 1024 / ctas_per_sm - 1024);
  const long long cap = per_cta - (long long)stream_smem_bytes(n_x, K, tl, steps, list_cap, 0);
  return cap > 0 ? int(cap & ~15LL) : 0;
}

void plan_stream_chunks(StreamLaunch& a, int sm_count) {
  // minimise waves x scenarios per CTA (ctas_per_sm CTAs resident per SM)
  sm_count *= std::max(1, a.ctas_per_sm);
  const int tiles = (a.n_u + a.K - 1) / a.K;
  long long best = -1;
  int best_n = 1;
  for (int nc = 1; nc <= a.M; ++nc) {
    const int chunk = (a.M + nc - 1) / nc;
    const int ncc = (a.M + chunk - 1) / chunk;
    const long long waves = (tiles * (long long)ncc + sm_count - 1) / sm_count;
    const long long cost = waves * chunk;
    if (best < 0 || cost < best) {
      best = cost;
      best_n = ncc;
    }
  }
  // then two scenarios per CTA when that plan is within 2 % of the cost:
  // half the partial K_hat slabs (each chunk writes one, finish_reduce reads
  // them all: 4.3 GB at 2869/512 with one scenario per CTA) and the producer
  // prefetches across the scenario boundary (1354/256: 12.96 against 13.05 ms
  // per tile kernel; 4 per CTA measured 13.14)
  for (int nc = (a.M + 1) / 2; nc < best_n; ++nc) {
    const int chunk = (a.M + nc - 1) / nc;
    if (chunk > 2) continue;
    const int ncc = (a.M + chunk - 1) / chunk;
    const long long waves = (tiles * (long long)ncc + sm_count - 1) / sm_count;
    if (waves * chunk * 50 <= best * 51) {
      best_n = ncc;
      break;
    }
  }
  a.chunk = (a.M + best_n - 1) / best_n;
  if (const char* e = std::getenv("BIPM_STREAM_CHUNK"))  // experiments: scenarios per CTA
    a.chunk = std::max(1, std::min(a.M, std::atoi(e)));
  a.nchunks = (a.M + a.chunk - 1) / a.chunk;
}

template <int K, int C>
static void launch_k(const StreamLaunch& a, cudaStream_t st) {
  const int tiles = (a.n_u + K - 1) / K;
  const size_t smem = stream_smem_bytes(a.n_x, K, a.tl, a.steps, a.list_cap, a.ring_bytes);
  cudaFuncSetAttribute(reduce_stream_kernel<K, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  reduce_stream_kernel<K, C><<<dim3(tiles, a.nchunks), C + 32, smem, st>>>(a);
  note_launch();
}

void launch_reduce_stream(const StreamLaunch& a, cudaStream_t st) {
  if (a.M <= 0) return;
  if (a.nq > kMaxQ) throw std::runtime_error("reduce_stream: too many accumulator registers");
  const int code = a.K * 1000 + a.consumers;
  switch (code) {
    case 1512: launch_k<1, 512>(a, st); break;
    case 2512: launch_k<2, 512>(a, st); break;
    case 4512: launch_k<4, 512>(a, st); break;
    case 8512: launch_k<8, 512>(a, st); break;
    case 16512: launch_k<16, 512>(a, st); break;
    case 32512: launch_k<32, 512>(a, st); break;
    case 1256: launch_k<1, 256>(a, st); break;
    case 2256: launch_k<2, 256>(a, st); break;
    case 4256: launch_k<4, 256>(a, st); break;
    case 8256: launch_k<8, 256>(a, st); break;
    case 1128: launch_k<1, 128>(a, st); break;
    case 2128: launch_k<2, 128>(a, st); break;
    case 4128: launch_k<4, 128>(a, st); break;
    default: throw std::runtime_error("reduce_stream: unsupported tile width / consumer count");
  }
  check_launch("reduce_stream");
}

void launch_kuu_sum(const double* kuu, long long stride, const int* row, const int* col, int nnz,
                    int M, int n_u, double* out, cudaStream_t st) {
  if (nnz <= 0 || M <= 0) return;
  kuu_sum_kernel<<<(nnz + 255) / 256, 256, 0, st>>>(kuu, stride, row, col, nnz, M, n_u, out);
  note_launch();
  check_launch("kuu_sum");
}

void launch_gather_values(const double* in, long long in_stride, const int* slot, int n,
                          double* out, long long out_stride, int M, cudaStream_t st) {
  const long long t = (long long)n * M;
  if (t <= 0) return;
  gather_values_kernel<<<int((t + 255) / 256), 256, 0, st>>>(in, in_stride, slot, n, out,
                                                             out_stride, M);
  note_launch();
  check_launch("gather_values");
}

}  // namespace bipm
