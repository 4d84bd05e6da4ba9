// Physics drivers on the device: per-time contour forward solves (solve_forward /
// solve_forward_batch, forward.cpp:75-198), quadrature recombination in basis form
// (phi(t) = 2 Re U c, c_j = sum_k w_k qhat_k y_kj; talbot.cpp:82-94 + forward.cpp:104-115),
// adjoint solves (jacobian.cpp:47-55) and the adjoint-state Jacobian assembly
// (sensitivity_row_conductivity / _storativity, jacobian.cpp:57-125, FD form of SURVEY
// App. A) for all source/receiver pairs of a time slice.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "drivers.hpp"
#include "lt_internal.hpp"
#include "stencil.cuh"
#include "talbot_host.hpp"

namespace lt {

thread_local std::vector<int> g_last_unconverged;

namespace {

constexpr int kT = 256;
using cd = std::complex<double>;

inline double2 d2(cd c) { return make_double2(c.real(), c.imag()); }

// heads[dst[b] + a] += 2 Re sum_j c[b][j] U_j[b][a]   (dst[b] < 0: item skipped)
__global__ void __launch_bounds__(kT) recombine_kernel(int64_t n, int B, int mc, const double2* const* __restrict__ Ucols,
                                                       const double2* __restrict__ c, const int64_t* __restrict__ dst,
                                                       double* __restrict__ heads) {
  LT_ITEM_BLOCK(B, b, cb);
  const int64_t a = (int64_t)cb * blockDim.x + threadIdx.x;
  if (a >= n || dst[b] < 0) return;
  double s = 0.0;
  for (int j = 0; j < mc; ++j) {
    const double2 cj = c[b * mc + j];
    const double2 u = Ucols[j][b * n + a];
    s += cj.x * u.x - cj.y * u.y;
  }
  heads[dst[b] + a] += 2.0 * s;
}

// drawdown[b][r] = sum_q w_q heads[b][idx_q]
__global__ void gather_points(int64_t n, int B, int n_pts, const double* __restrict__ heads, const int64_t* __restrict__ idx,
                              const double* __restrict__ w, const int* __restrict__ cnt, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * n_pts) return;
  const int b = t / n_pts, r = t % n_pts;
  double s = 0.0;
  for (int q = 0; q < cnt[r]; ++q) s += w[r * 8 + q] * heads[b * n + idx[r * 8 + q]];
  out[t] = s;
}

// predictions[s][r] = 2 Re sum_k w_k sum_q wq phi_{s,k}[idx_q]
// (cell_major fields: f[(k n + a) B + s], B = n_src + n_rec)
__global__ void predict_kernel(int64_t n, int n_src, int n_rec, int ns, const double2* __restrict__ fields,
                               const double2* __restrict__ w, const int64_t* __restrict__ idx, const double* __restrict__ wt,
                               const int* __restrict__ cnt, double* __restrict__ out, int cell_major) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_src * n_rec) return;
  const int s = t / n_rec, r = t % n_rec;
  const int B = n_src + n_rec;
  double2 acc = make_double2(0.0, 0.0);
  for (int k = 0; k < ns; ++k) {
    double2 v = make_double2(0.0, 0.0);
    for (int q = 0; q < cnt[r]; ++q) {
      const int64_t a = idx[r * 8 + q];
      const double2 fv = cell_major ? fields[((int64_t)k * n + a) * B + s] : fields[((int64_t)s * ns + k) * n + a];
      v = cadd(v, cscale(fv, wt[r * 8 + q]));
    }
    acc = cadd(acc, cmul(w[k], v));
  }
  out[t] = 2.0 * acc.x;
}

// rhs[item*n + idx] += w for the sparse point weights of each item (zeroed beforehand)
__global__ void scatter_points(int64_t n, int n_items, const int64_t* __restrict__ idx, const double* __restrict__ w,
                               const int* __restrict__ cnt, double2* __restrict__ rhs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_items * 8) return;
  const int it = t / 8, q = t % 8;
  if (q >= cnt[it]) return;
  rhs[(int64_t)it * n + idx[it * 8 + q]].x += w[it * 8 + q];
}

__global__ void real_to_complex(int64_t n, const double* __restrict__ x, double2* __restrict__ y) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) y[a] = make_double2(x[a], 0.0);
}

// ---- Jacobian assembly -----------------------------------------------------------------
// J_k[(s,r), a] = 2 Re sum_k w_k sum_{f in faces(a)} dT_f/dln k_a (phi_a - phi_b)(psi_a - psi_b)
// J_S[(s,r), a] = 2 Re sum_k w_k z_k^p S_a h^d phi_a psi_a
// A CTA owns TC consecutive cells of one row and all (source-block x receiver-block)
// register tiles.  Per shift k, every field value at the tile (centre) and its 2d face
// neighbours is loaded once, the 2d weighted face differences and the storativity term of
// all sources (P) and receivers (Q) are staged in shared memory, and every thread
// accumulates its SB x RB tile of Re(P Q) for one cell over the 2d+1 stages.
constexpr int SB = 4;
constexpr int RB = 8;

template <int DIM>
__global__ void __launch_bounds__(kT, 2) jacobian_kernel(LevelView L, const double* __restrict__ kappa,
                                                      const double* __restrict__ stor, double hd, double face_scale,
                                                      const double2* __restrict__ fields, int n_src, int n_rec, int ns,
                                                      const double2* __restrict__ w, const double2* __restrict__ wz,
                                                      int TC, int tiles_x, int nsub_r, int nsub_total,
                                                      double* __restrict__ Jk, double* __restrict__ Js, int64_t ldj) {
  constexpr int NF = 2 * DIM + 1;  // faces + storativity stage
  extern __shared__ double2 smem[];
  const int n_items = n_src + n_rec;
  double2* P = smem;                                    // [2 DIM][n_src][TC]
  double2* Q = smem + (size_t)2 * DIM * n_src * TC;     // [2 DIM][n_rec][TC]
  double* wt = reinterpret_cast<double*>(Q + (size_t)2 * DIM * n_rec * TC);  // [NF][TC]
  int64_t* nb = reinterpret_cast<int64_t*>(wt + NF * TC);             // [2 DIM][TC] neighbour index or -1
  const int64_t n = L.n;
  // tile -> (row, x offset); cells of one tile are consecutive in x
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x;
  const int64_t row = tile / tiles_x;  // k * ny + j
  const int i0 = tx * TC;
  const int ncell = min(TC, L.nx - i0);
  const int64_t a0 = row * L.nx + i0;
  const int j = (int)(row % L.ny);
  const int kz = (int)(row / L.ny);
  const int tid = threadIdx.x;
  const int c = tid % TC;
  const int sub = tid / TC;
  const bool owner = sub < nsub_total && c < ncell;
  const int s0 = owner ? (sub / nsub_r) * SB : 0;
  const int r0 = owner ? (sub % nsub_r) * RB : 0;

  if (tid < NF * TC) {
    const int f = tid / TC, cc = tid % TC;
    double wv = 0.0;
    int64_t nbi = -1;
    if (cc < ncell) {
      const int64_t a = a0 + cc;
      if (f == 2 * DIM) {
        wv = stor[a] * hd;
      } else {
        const int d = f >> 1, hi = f & 1;
        const int coord = d == 0 ? i0 + cc : (d == 1 ? j : kz);
        const int ext = d == 0 ? L.nx : (d == 1 ? L.ny : L.nz);
        const int64_t stride = d == 0 ? 1 : (d == 1 ? (int64_t)L.nx : (int64_t)L.nx * L.ny);
        const double ka = kappa[a];
        const bool boundary = hi ? coord == ext - 1 : coord == 0;
        if (boundary) {
          wv = 2.0 * ka * face_scale;  // dT/dln k_a = T = 2 k_a h^(d-2); ghost value 0
        } else {
          nbi = hi ? a + stride : a - stride;
          const double kb = kappa[nbi];
          const double T = 2.0 * ka * kb / (ka + kb) * face_scale;
          wv = T * kb / (ka + kb);
        }
      }
    }
    wt[f * TC + cc] = wv;
    if (f < 2 * DIM) nb[f * TC + cc] = nbi;
  }

  __syncthreads();
  // phase 0: kappa block over the 2d face stages; phase 1: storativity block (centre stage).
  // Two phases keep one SB x RB accumulator tile per thread (2 CTAs per SM).
  for (int phase = 0; phase < (Js ? 2 : 1); ++phase) {
    double acc[SB][RB];
#pragma unroll
    for (int i = 0; i < SB; ++i)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[i][q] = 0.0;
    const int nstage = phase == 0 ? 2 * DIM : 1;
    for (int k = 0; k < ns; ++k) {
      const double2 wk = w[k], wzk = wz[k];
      // stage: one centre (+ 2d neighbour) loads per (item, cell)
      for (int e = tid; e < n_items * TC; e += blockDim.x) {
        const int it = e / TC, cc = e % TC;
        const double2* fld = fields + ((int64_t)it * ns + k) * n;
        const double2 fa = cc < ncell ? fld[a0 + cc] : make_double2(0.0, 0.0);
        if (phase == 0) {
          double2 fn[2 * DIM];
#pragma unroll
          for (int f = 0; f < 2 * DIM; ++f) {
            const int64_t q = cc < ncell ? nb[f * TC + cc] : -1;
            fn[f] = q >= 0 ? fld[q] : make_double2(0.0, 0.0);
          }
          if (it < n_src) {
#pragma unroll
            for (int f = 0; f < 2 * DIM; ++f)
              P[((size_t)f * n_src + it) * TC + cc] = cscale(cmul(wk, csub(fa, fn[f])), wt[f * TC + cc]);
          } else {
            const int r = it - n_src;
#pragma unroll
            for (int f = 0; f < 2 * DIM; ++f) Q[((size_t)f * n_rec + r) * TC + cc] = csub(fa, fn[f]);
          }
        } else {
          if (it < n_src) P[(size_t)it * TC + cc] = cscale(cmul(wzk, fa), wt[2 * DIM * TC + cc]);
          else Q[(size_t)(it - n_src) * TC + cc] = fa;
        }
      }
      __syncthreads();
      if (owner) {
#pragma unroll 1
        for (int f = 0; f < nstage; ++f) {
          double2 pv[SB];
#pragma unroll
          for (int i = 0; i < SB; ++i)
            pv[i] = (s0 + i < n_src) ? P[((size_t)f * n_src + s0 + i) * TC + c] : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const double2 qv = (r0 + q < n_rec) ? Q[((size_t)f * n_rec + r0 + q) * TC + c] : make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < SB; ++i) acc[i][q] = fma(pv[i].x, qv.x, fma(-pv[i].y, qv.y, acc[i][q]));
          }
        }
      }
      __syncthreads();
    }
    if (owner) {
      double* Jout = phase == 0 ? Jk : Js;
      const int64_t a = a0 + c;
#pragma unroll
      for (int i = 0; i < SB; ++i) {
        if (s0 + i >= n_src) continue;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          if (r0 + q >= n_rec) continue;
          const int64_t rowj = (int64_t)(s0 + i) * n_rec + (r0 + q);
          Jout[rowj * ldj + a] = 2.0 * acc[i][q];
        }
      }
    }
  }
}

// ---- Jacobian on the FP64 tensor cores (mma.sync m8n8k4 .f64) ------------------------------
// Per cell a the kappa and storativity rows are small real GEMMs.  With the 2d+1 points of the
// cell (centre, face neighbours b_f) and the arrow transform of the source fields
//   A_0 = w_k sum_f wt_f (phi_a - phi_bf),  A_f = -w_k wt_f (phi_a - phi_bf),
// sum_f wt_f (phi_a - phi_bf)(psi_a - psi_bf) = sum_p A_p psi_p, so
//   J_k[s, r] = 2 Re sum_{k, p} A_{k,p}[s] psi_{k,p}[r],   J_S[s, r] = 2 Re sum_k wz_k S_a h^d phi_a psi_a
// = real GEMMs over K = (shift, point, re/im) whose B operand is the raw receiver field (no
// difference pass for the receivers).  A persistent CTA walks tasks = (tile of 2 cells of a
// row, pair of shifts), warp-specialised:
//   copy warp 16   : bulk-copies each task's raw fields (all items at the tile's 12 points,
//                     one contiguous B x 16-byte run per (shift, point) of the cell-major field
//                     array) into a 4-deep ring, gated only by the ring's empty barriers (a
//                     dedicated warp: issuing from a transform warp tied each refill to that
//                     warp's transform of the next task, ~30% of the kernel's time);
//   producer warps 8-15: the arrow transform of the 16 sources into mma A fragments
//                     (3 buffers; 4 lanes per (cell, shift, source), faces split);
//   consumer warps 0-7: warp = (cell, 16 receivers): 2 x 2 accumulator tiles per block.
// mbarriers hand the stages over; J is written after a tile's last shift pair.
// Requires n_src <= 16 and n_rec <= 64.
constexpr int JW_TC = 2;  // cells per tile
constexpr int JW_SMAX = 16, JW_RMAX = 64;
constexpr int JW_NRAW = 4;
constexpr int JW_CONS = 8, JW_PROD = 8;
constexpr int JW_NA = 3;  // A-fragment buffers
constexpr int JW_THREADS = 32 * (JW_CONS + JW_PROD + 1);  // + the copy warp

template <int DIM>
struct JwGeom {
  static constexpr int NPC = 2 * DIM + 1;          // points per cell
  static constexpr int NCH = DIM == 3 ? 36 : 24;   // B-item chunks per ring slot (two TMA boxes)
  static constexpr int KS = NPC;                    // K steps per shift pair (2 NPC 2 / 4)
};

// A ring slot holds two TMA boxes of the cell-major field array (x = cells of the row):
//   box A: shifts kp..kp+1 x rows j-1..j+1 x cells i0-1..i0+2       (24 chunks, [s2][y][x])
//   box B: shifts kp..kp+1 x planes kz-1..kz+1 x cells i0..i0+1     (12 chunks, [s2][z][x], 3-D)
// each chunk = all B items of one (shift, cell); out-of-domain cells and the padding shift
// arrive as zeros (TMA out-of-bounds fill).  Chunk of cell c's point p (0 centre, 1..6 faces):
template <int DIM>
__device__ __forceinline__ int jw_chunk(int s2, int c, int p) {
  switch (p) {
    case 0: return (s2 * 3 + 1) * 4 + c + 1;
    case 1: return (s2 * 3 + 1) * 4 + c;
    case 2: return (s2 * 3 + 1) * 4 + c + 2;
    case 3: return (s2 * 3 + 0) * 4 + c + 1;
    case 4: return (s2 * 3 + 2) * 4 + c + 1;
    case 5: return 24 + (s2 * 3 + 0) * 2 + c;
    default: return 24 + (s2 * 3 + 2) * 2 + c;
  }
}

// ring slot layout (complex units): box A at 0, box B at jw_offb(B); both 128-byte aligned
__host__ __device__ inline int jw_offb(int B) { return ((24 * B * 16 + 127) / 128) * 8; }
template <int DIM>
__host__ __device__ inline int jw_slot(int B) {
  return (((jw_offb(B) + (DIM == 3 ? 12 * B : 0)) * 16 + 127) / 128) * 8;
}

template <int DIM>
size_t jw_smem(int B) {
  using G = JwGeom<DIM>;
  return sizeof(double2) * JW_NRAW * (size_t)jw_slot<DIM>(B)        // raw ring
         + sizeof(double) * JW_NA * JW_TC * 2 * (G::KS + 1) * 32     // A fragments [buf][cell][mt][ks][lane]
         + sizeof(double) * 2 * JW_TC * G::NPC;                      // weights [tile parity]
}

__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
#ifdef LT_JAC_DFMA
  // A/B build only (scripts/jac_ab.py): the same m8n8k4 product on the DFMA pipe.  Lane (g, q)
  // holds A[g][q], B[q][g] and C[g][2q .. 2q+1]; it gathers A[g][0..3] and B[0..3][2q .. 2q+1]
  // from the owning lanes.
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double ak = __shfl_sync(0xffffffff, a, g * 4 + k);
    const double b0 = __shfl_sync(0xffffffff, b, (2 * q) * 4 + k);
    const double b1 = __shfl_sync(0xffffffff, b, (2 * q + 1) * 4 + k);
    c[0] = fma(ak, b0, c[0]);
    c[1] = fma(ak, b1, c[1]);
  }
#else
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
#endif
}
__device__ __forceinline__ uint32_t jw_s(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   jw_s(dst)),
               "l"(src), "r"(bytes), "r"(jw_s(bar))
               : "memory");
}
__device__ __forceinline__ void jw_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(jw_s(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void jw_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(jw_s(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void jw_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(jw_s(b)) : "memory");
}
__device__ __forceinline__ void jw_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(jw_s(b)), "r"(parity)
        : "memory");
  } while (!ok);
}

template <int DIM>
__global__ void __launch_bounds__(JW_THREADS, 1) jacobian_mma_kernel(
    const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, LevelView L,
    const double* __restrict__ kappa, const double* __restrict__ stor, double hd, double face_scale, int n_src, int n_rec,
    int ns, const double2* __restrict__ w,
    const double2* __restrict__ wz, double* __restrict__ Jk, double* __restrict__ Js, int64_t ldj, int ntiles) {
  using G = JwGeom<DIM>;
  constexpr int NPC = G::NPC, NCH = G::NCH, KS = G::KS;
  constexpr int AF = JW_TC * 2 * (KS + 1) * 32;  // doubles per A-fragment buffer
  extern __shared__ __align__(128) unsigned char jsm[];
  __shared__ __align__(8) uint64_t raw_full[JW_NRAW], raw_empty[JW_NRAW], a_full[JW_NA], a_empty[JW_NA];
  const int B = n_src + n_rec;
  double2* raw = reinterpret_cast<double2*>(jsm);                       // [JW_NRAW][NCH][B]
  const int SLOT = jw_slot<DIM>(B), OFFB = jw_offb(B);
  auto chunk = [&](int ch) { return ch < 24 ? ch * B : OFFB + (ch - 24) * B; };  // complex offset in a slot
  double* Af = reinterpret_cast<double*>(raw + JW_NRAW * SLOT);       // [JW_NA][AF]
  double* wts = Af + JW_NA * AF;  // [tile parity][TC][NPC] (p = 0: S h^d)
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const int tiles_x = (L.nx + JW_TC - 1) / JW_TC;
  const int64_t n = L.n, plane = (int64_t)L.nx * L.ny;
  if ((int)blockIdx.x >= ntiles) return;
  const int npair = (ns + 1) / 2;
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int T = my_tiles * npair;
  struct TileXY {
    int i0, j, kz;
  };
  // tile order: x segments fastest, then YB rows, then planes, then blocks of YB rows, so the
  // CTAs in flight at any time cover YB rows x ~all planes' neighbours: the y and z face
  // neighbours of a tile are loaded by concurrently running tiles (L2 hits, not HBM re-reads)
  const int YB = (L.ny % 4 == 0) ? 4 : ((L.ny % 2 == 0) ? 2 : 1);
  auto tile_at = [&](int t) {
    const int tile = (int)blockIdx.x + (t / npair) * (int)gridDim.x;
    const int tx = tile % tiles_x, r = tile / tiles_x;
    const int yi = r % YB, r2 = r / YB;
    const int kz = r2 % L.nz, yb = r2 / L.nz;
    return TileXY{tx * JW_TC, yb * YB + yi, kz};
  };
  if (tid == 0) {
    for (int q = 0; q < JW_NRAW; ++q) {
      jw_init(&raw_full[q], 1);
      jw_init(&raw_empty[q], JW_CONS + JW_PROD);
    }
    for (int q = 0; q < JW_NA; ++q) {
      jw_init(&a_full[q], JW_PROD);
      jw_init(&a_empty[q], JW_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wc == JW_CONS + JW_PROD) {
    // ------------------------------- copy warp -------------------------------------------
    // task t's two boxes into slot t % JW_NRAW once every consumer and producer warp has
    // released the slot's previous task (t - JW_NRAW)
    if (lane == 0) {
      for (int t = 0; t < T; ++t) {
        const int slot = t % JW_NRAW;
        if (t >= JW_NRAW) jw_wait(&raw_empty[slot], (uint32_t)(((t - JW_NRAW) / JW_NRAW) & 1));
        const TileXY g = tile_at(t);
        const int kp = (t % npair) * 2;
        double2* dst = raw + slot * SLOT;
        const uint32_t ca = (uint32_t)B * 16u;
        jw_expect(&raw_full[slot], 24u * ca + (DIM == 3 ? 12u * ca : 0u));
        tma5(dst, &mA, 0, g.i0 - 1, g.j - 1, g.kz, kp, &raw_full[slot]);
        if (DIM == 3) tma5(dst + OFFB, &mB, 0, g.i0, g.j, g.kz - 1, kp, &raw_full[slot]);
      }
    }
  } else if (wc >= JW_CONS) {
    // ------------------------------- producers -------------------------------------------
    const int ptid = tid - 32 * JW_CONS;
    // face / storativity weights of tile u into wts[u & 1] (loads issued a tile ahead of use)
    auto weights = [&](int u) {
      if (ptid >= JW_TC * NPC || u * npair >= T) return;
      const TileXY g = tile_at(u * npair);
      const int c = ptid / NPC, p = ptid % NPC;
      const int i = g.i0 + c;
      double wv = 0.0;
      if (i < L.nx) {
        const int64_t a = ((int64_t)g.kz * L.ny + g.j) * L.nx + i;
        if (p == 0) {
          wv = stor[a] * hd;
        } else {
          const int f = p - 1, d = f >> 1, hi = f & 1;
          const int coord = d == 0 ? i : (d == 1 ? g.j : g.kz);
          const int ext = d == 0 ? L.nx : (d == 1 ? L.ny : L.nz);
          const int64_t stride = d == 0 ? 1 : (d == 1 ? (int64_t)L.nx : plane);
          const double ka = kappa[a];
          if (hi ? coord == ext - 1 : coord == 0) {
            wv = 2.0 * ka * face_scale;  // dT/dln k_a = T = 2 k_a h^(d-2); ghost value 0
          } else {
            const double kb = kappa[hi ? a + stride : a - stride];
            const double Tf = 2.0 * ka * kb / (ka + kb) * face_scale;
            wv = Tf * kb / (ka + kb);
          }
        }
      }
      wts[(u & 1) * JW_TC * NPC + c * NPC + p] = wv;
    };
    weights(0);
    for (int t = 0; t < T; ++t) {
      const int kp = (t % npair) * 2;
      const double* wt = wts + ((t / npair) & 1) * JW_TC * NPC;
      if (t % npair == 0) {
        // this tile's weights (stored a tile ago) are visible after the producers' barrier; the
        // next tile's go into the other half (its previous user, tile - 1, is finished)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * JW_PROD) : "memory");
        weights(t / npair + 1);
      }
      jw_wait(&raw_full[t % JW_NRAW], (uint32_t)((t / JW_NRAW) & 1));
      if (t >= JW_NA) jw_wait(&a_empty[t % JW_NA], (uint32_t)(((t - JW_NA) / JW_NA) & 1));
      // arrow transform: 4 lanes per (cell, shift of the pair, source), faces p - 1 = part mod 4
      {
        const double2* rw = raw + (t % JW_NRAW) * SLOT;
        double* Ab = Af + (t % JW_NA) * AF;
        const int combo = ptid >> 2, part = ptid & 3;
        const int s = combo % JW_SMAX, s2 = (combo / JW_SMAX) % 2, c = combo / (2 * JW_SMAX);
        const int k = kp + s2;
        const bool live = s < n_src && k < ns;
        // w == nullptr: the source fields already carry w_k (expand), wz then holds z_k or 1
        const double2 wk = live ? (w ? w[k] : make_double2(1.0, 0.0)) : make_double2(0.0, 0.0);
        const double2* R = rw + min(s, B - 1);
        const double2 pa = R[chunk(jw_chunk<DIM>(s2, c, 0))];
        const int mt = s >> 3, lrow = (s & 7) * 4;
        double* Ac = Ab + (c * 2 + mt) * (KS + 1) * 32;
        auto put = [&](int p, double2 v) {  // A'[s][K], K = (s2 NPC + p) 2 + comp (re, -im)
          const int K0 = (s2 * NPC + p) * 2;
          Ac[(K0 >> 2) * 32 + lrow + (K0 & 3)] = v.x;
          Ac[((K0 + 1) >> 2) * 32 + lrow + ((K0 + 1) & 3)] = -v.y;
        };
        double2 a0 = make_double2(0.0, 0.0);
#pragma unroll
        for (int p = 1; p < NPC; ++p) {
          if ((p - 1) % 4 != part) continue;
          const double2 d = live ? cscale(csub(pa, R[chunk(jw_chunk<DIM>(s2, c, p))]), wt[c * NPC + p]) : make_double2(0.0, 0.0);
          a0 = cadd(a0, d);
          put(p, w ? cmul(wk, make_double2(-d.x, -d.y)) : make_double2(-d.x, -d.y));
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          a0.x += __shfl_xor_sync(0xffffffffu, a0.x, o);
          a0.y += __shfl_xor_sync(0xffffffffu, a0.y, o);
        }
        if (part == 0) put(0, w ? cmul(wk, a0) : a0);
        if (part == 1) {  // storativity block: K = s2 2 + comp in step KS
          const double2 As = live ? cmul(wz[k], cscale(pa, wt[c * NPC])) : make_double2(0.0, 0.0);
          Ac[KS * 32 + lrow + s2 * 2] = As.x;
          Ac[KS * 32 + lrow + s2 * 2 + 1] = -As.y;
        }
      }
      __syncwarp();
      if (lane == 0) {
        jw_arrive(&a_full[t % JW_NA]);
        jw_arrive(&raw_empty[t % JW_NRAW]);
      }
    }
  } else {
    // ------------------------------- consumers -------------------------------------------
    // warp -> receivers wc*8 .. +7 of both cells (the two cells' J entries of one row are
    // adjacent: one 16-byte store)
    const int kq = lane & 3, rl = lane >> 2;
    const int rcol = n_src + min(wc * 8 + rl, n_rec - 1);
    double accK[2][2][2], accS[2][2][2];  // [cell][m tile][2]
    for (int t = 0; t < T; ++t) {
      const TileXY g = tile_at(t);
      if (t % npair == 0) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) accK[c][mt][0] = accK[c][mt][1] = accS[c][mt][0] = accS[c][mt][1] = 0.0;
      }
      jw_wait(&raw_full[t % JW_NRAW], (uint32_t)((t / JW_NRAW) & 1));
      jw_wait(&a_full[t % JW_NA], (uint32_t)((t / JW_NA) & 1));
      const double2* rw = raw + (t % JW_NRAW) * SLOT;
      const double* Ab = Af + (t % JW_NA) * AF;
      {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double* Ac = Ab + c * 2 * (KS + 1) * 32;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const int K = ks * 4 + kq, comp = K & 1, s2 = K / (2 * NPC), p = (K >> 1) % NPC;
            const double bv = reinterpret_cast<const double*>(rw + chunk(jw_chunk<DIM>(s2, c, p)))[2 * rcol + comp];
            dmma(accK[c][0], Ac[ks * 32 + lane], bv);
            dmma(accK[c][1], Ac[(KS + 1) * 32 + ks * 32 + lane], bv);
          }
          {  // storativity: K = s2 2 + comp at the centre point
            const int s2 = kq >> 1, comp = kq & 1;
            const double bv = reinterpret_cast<const double*>(rw + chunk(jw_chunk<DIM>(s2, c, 0)))[2 * rcol + comp];
            dmma(accS[c][0], Ac[KS * 32 + lane], bv);
            dmma(accS[c][1], Ac[(KS + 1) * 32 + KS * 32 + lane], bv);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        jw_arrive(&a_empty[t % JW_NA]);
        jw_arrive(&raw_empty[t % JW_NRAW]);
      }
      if (t % npair == npair - 1) {
        const int64_t a = ((int64_t)g.kz * L.ny + g.j) * L.nx + g.i0;
        const bool both = g.i0 + 1 < L.nx;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int s = mt * 8 + (lane >> 2);
          if (s >= n_src) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wc * 8 + (lane & 3) * 2 + h;
            if (r >= n_rec) continue;
            const int64_t o = ((int64_t)s * n_rec + r) * ldj + a;
            double* pk = Jk + o;
            if (both && ((reinterpret_cast<uintptr_t>(pk) & 15) == 0)) {
              *reinterpret_cast<double2*>(pk) = make_double2(2.0 * accK[0][mt][h], 2.0 * accK[1][mt][h]);
            } else {
              pk[0] = 2.0 * accK[0][mt][h];
              if (both) pk[1] = 2.0 * accK[1][mt][h];
            }
            if (Js) {
              double* ps = Js + o;
              if (both && ((reinterpret_cast<uintptr_t>(ps) & 15) == 0)) {
                *reinterpret_cast<double2*>(ps) = make_double2(2.0 * accS[0][mt][h], 2.0 * accS[1][mt][h]);
              } else {
                ps[0] = 2.0 * accS[0][mt][h];
                if (both) ps[1] = 2.0 * accS[1][mt][h];
              }
            }
          }
        }
      }
    }
  }
}

// ---- Jacobian on the FP64 tensor cores, 4-cell tiles -----------------------------------------
// The same GEMM formulation as jacobian_mma_kernel (arrow transform of the sources, raw receiver
// fields as the B operand), with a task = (4 consecutive cells of a row, pair of shifts):
//  * the halo costs 44 chunks per 8 (cell, shift) units (centre row i0-1..i0+4, rows j-1 / j+1
//    and planes kz-1 / kz+1 over i0..i0+3: five TMA boxes, no corner cells) instead of 36 per 4:
//    5.5x instead of 9x the field bytes from L2 per cell and shift;
//  * every lane ends a tile holding the 4 cells of each of its (s, r) entries and writes them as
//    one 32-byte store (STG.256) -- full L2 sectors, where 2-cell tiles wrote half sectors
//    (ncu: 16 of 32 bytes per sector used), half the store transactions;
//  * a dedicated copy warp keeps the 3-deep ring full, gated only by its empty barriers.
// Warps: 0-7 consumers (8 receivers x 4 cells x 16 sources each), 8-11 producers (arrow
// transform, one lane per (cell, shift, source)), 12 the copy warp (13 warps: <= 4 per SM
// sub-partition, so 128 registers per thread).  Needs nx % 4 == 0,
// n_src <= 16, n_rec <= 64 and 32-byte aligned J rows (checked by the caller).
constexpr int J4_TC = 4;
// faces-only K (B operand psi_f - psi_a formed by the consumers; no centre column): 1/8 fewer
// DMMA steps per shift pair than the arrow transform with its centre column (47.4 vs 49.6 ms per
// 128^3 slice)
constexpr int J4_NRAW = 3, J4_NA = 3;
constexpr int J4_CONS = 8, J4_PROD = 4;
constexpr int J4_THREADS = 32 * (J4_CONS + J4_PROD + 1);

// slot regions (complex offsets, each 128-byte aligned): C = centre row, 6 cells x 2 shifts;
// then 4-cell x 2-shift boxes S (row j-1), N (row j+1), D (plane kz-1), U (plane kz+1)
__host__ __device__ inline int j4_rnd(int cplx) { return ((cplx * 16 + 127) / 128) * 8; }
__host__ __device__ inline int j4_offC() { return 0; }
__host__ __device__ inline int j4_offF(int B, int f) { return j4_rnd(12 * B) + f * j4_rnd(8 * B); }  // f: 0 S 1 N 2 D 3 U
template <int DIM>
__host__ __device__ inline int j4_slot(int B) { return j4_offF(B, DIM == 3 ? 4 : 2); }

template <int DIM>
size_t j4_smem(int B) {
  constexpr int NPC = 2 * DIM + 1, KS = NPC - 1;  // faces-only K steps (+1: the storativity step)
  return sizeof(double2) * J4_NRAW * (size_t)j4_slot<DIM>(B)      // raw ring
         + sizeof(double) * J4_NA * J4_TC * 2 * ((KS + 1) * 32 + 1) // A fragments [buf][cell][mt][ks][lane] (+pad)
         + sizeof(double) * 2 * J4_TC * NPC;                       // weights [tile parity][cell][point]
}

// complex offset in a slot of cell c's point p (0 centre, 1 W, 2 E, 3 S, 4 N, 5 D, 6 U), shift s2
__device__ __forceinline__ int j4_at(int B, int s2, int c, int p) {
  switch (p) {
    case 0: return (s2 * 6 + c + 1) * B;
    case 1: return (s2 * 6 + c) * B;
    case 2: return (s2 * 6 + c + 2) * B;
    default: return j4_offF(B, p - 3) + (s2 * 4 + c) * B;
  }
}

// 32-byte store with an L2 evict-first policy: J (34 GB per 128^3 slice) streams through L2
// without evicting the field planes the neighbouring tiles still read
__device__ __forceinline__ void stg256(double* p, double a, double b, double c, double d, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d), "l"(pol)
               : "memory");
}

template <int DIM>
__global__ void __launch_bounds__(J4_THREADS, 1) jacobian_mma4_kernel(
    const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mF, LevelView L,
    const double* __restrict__ kappa, const double* __restrict__ stor, double hd, double face_scale, int n_src,
    int n_rec, int ns, const double2* __restrict__ wz, double* __restrict__ Jk, double* __restrict__ Js, int64_t ldj,
    int ntiles) {
  constexpr int NPC = 2 * DIM + 1;
  // faces only: B operand psi_f - psi_a formed by the consumers, K per shift pair 4 NF
  constexpr int NF = NPC - 1, KS = NF;
  constexpr int MTS = (KS + 1) * 32 + 1;  // doubles per (cell, m tile) fragment block (+1: bank spread)
  constexpr int AF = J4_TC * 2 * MTS;      // doubles per A-fragment buffer
  extern __shared__ __align__(128) unsigned char jsm[];
  __shared__ __align__(8) uint64_t raw_full[J4_NRAW], raw_empty[J4_NRAW], a_full[J4_NA], a_empty[J4_NA];
  const int B = n_src + n_rec;
  const int SLOT = j4_slot<DIM>(B);
  double2* raw = reinterpret_cast<double2*>(jsm);
  double* Af = reinterpret_cast<double*>(raw + J4_NRAW * SLOT);
  double* wts = Af + J4_NA * AF;
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const int tiles_x = L.nx / J4_TC;
  const int64_t plane = (int64_t)L.nx * L.ny;
  if ((int)blockIdx.x >= ntiles) return;
  const int npair = (ns + 1) / 2;
  const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int T = my_tiles * npair;
  struct TileXY {
    int i0, j, kz;
  };
  // x segments fastest, then YB rows, then planes, then blocks of YB rows: the tiles in flight
  // at any time share their y and z neighbours through L2
  const int YB = (L.ny % 4 == 0) ? 4 : ((L.ny % 2 == 0) ? 2 : 1);
  auto tile_at = [&](int t) {
    const int tile = (int)blockIdx.x + (t / npair) * (int)gridDim.x;
    const int tx = tile % tiles_x, r = tile / tiles_x;
    const int yi = r % YB, r2 = r / YB;
    const int kz = r2 % L.nz, yb = r2 / L.nz;
    return TileXY{tx * J4_TC, yb * YB + yi, kz};
  };
  if (tid == 0) {
    for (int q = 0; q < J4_NRAW; ++q) {
      jw_init(&raw_full[q], 1);
      jw_init(&raw_empty[q], J4_CONS + J4_PROD);
    }
    for (int q = 0; q < J4_NA; ++q) {
      jw_init(&a_full[q], J4_PROD);
      jw_init(&a_empty[q], J4_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wc == J4_CONS + J4_PROD) {
    // ------------------------------- copy warp -------------------------------------------
    if (lane == 0) {
      const uint32_t ca = (uint32_t)B * 16u;
      for (int t = 0; t < T; ++t) {
        const int slot = t % J4_NRAW;
        if (t >= J4_NRAW) jw_wait(&raw_empty[slot], (uint32_t)(((t - J4_NRAW) / J4_NRAW) & 1));
        const TileXY g = tile_at(t);
        const int kp = (t % npair) * 2;
        double2* dst = raw + slot * SLOT;
        jw_expect(&raw_full[slot], (12u + (DIM == 3 ? 32u : 16u)) * ca);
        tma5(dst + j4_offC(), &mC, 0, g.i0 - 1, g.j, g.kz, kp, &raw_full[slot]);
        tma5(dst + j4_offF(B, 0), &mF, 0, g.i0, g.j - 1, g.kz, kp, &raw_full[slot]);
        tma5(dst + j4_offF(B, 1), &mF, 0, g.i0, g.j + 1, g.kz, kp, &raw_full[slot]);
        if (DIM == 3) {
          tma5(dst + j4_offF(B, 2), &mF, 0, g.i0, g.j, g.kz - 1, kp, &raw_full[slot]);
          tma5(dst + j4_offF(B, 3), &mF, 0, g.i0, g.j, g.kz + 1, kp, &raw_full[slot]);
        }
      }
    }
  } else if (wc >= J4_CONS) {
    // ------------------------------- producers -------------------------------------------
    const int ptid = tid - 32 * J4_CONS;
    // face / storativity weights of tile u into wts[u & 1]
    auto weights = [&](int u) {
      if (ptid >= J4_TC * NPC || u * npair >= T) return;
      const TileXY g = tile_at(u * npair);
      const int c = ptid / NPC, p = ptid % NPC;
      const int i = g.i0 + c;
      const int64_t a = ((int64_t)g.kz * L.ny + g.j) * L.nx + i;
      double wv;
      if (p == 0) {
        wv = stor[a] * hd;
      } else {
        const int f = p - 1, d = f >> 1, hi = f & 1;
        const int coord = d == 0 ? i : (d == 1 ? g.j : g.kz);
        const int ext = d == 0 ? L.nx : (d == 1 ? L.ny : L.nz);
        const int64_t stride = d == 0 ? 1 : (d == 1 ? (int64_t)L.nx : plane);
        const double ka = kappa[a];
        if (hi ? coord == ext - 1 : coord == 0) {
          wv = 2.0 * ka * face_scale;  // dT/dln k_a = T = 2 k_a h^(d-2); ghost value 0
        } else {
          const double kb = kappa[hi ? a + stride : a - stride];
          const double Tf = 2.0 * ka * kb / (ka + kb) * face_scale;
          wv = Tf * kb / (ka + kb);
        }
      }
      wts[(u & 1) * J4_TC * NPC + c * NPC + p] = wv;
    };
    weights(0);
    // one lane per (cell, shift of the pair, source)
    const int combo = ptid;
    const int s = combo % JW_SMAX, s2 = (combo / JW_SMAX) % 2, c = combo / (2 * JW_SMAX);
    const int mt = s >> 3, lrow = (s & 7) * 4;
    for (int t = 0; t < T; ++t) {
      const int kp = (t % npair) * 2;
      const double* wt = wts + ((t / npair) & 1) * J4_TC * NPC;
      if (t % npair == 0) {
        // tile u's weights (stored a tile ago) are visible after this barrier; tile u + 1's go
        // into the other half (its previous user, tile u - 1, is finished)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * J4_PROD) : "memory");
        weights(t / npair + 1);
      }
      jw_wait(&raw_full[t % J4_NRAW], (uint32_t)((t / J4_NRAW) & 1));
      if (t >= J4_NA) jw_wait(&a_empty[t % J4_NA], (uint32_t)(((t - J4_NA) / J4_NA) & 1));
      {
        const double2* rw = raw + (t % J4_NRAW) * SLOT;
        double* Ac = Af + (t % J4_NA) * AF + (c * 2 + mt) * MTS;
        const int k = kp + s2;
        const bool live = s < n_src && k < ns;
        const double2* R = rw + min(s, B - 1);
        const double2 pa = R[j4_at(B, s2, c, 0)];
        auto put = [&](int p, double2 v) {  // A'[s][K], K = (s2 NPC + p) 2 + comp (re, -im)
          const int K0 = (s2 * NF + p - 1) * 2;
          Ac[(K0 >> 2) * 32 + lrow + (K0 & 3)] = v.x;
          Ac[((K0 + 1) >> 2) * 32 + lrow + ((K0 + 1) & 3)] = -v.y;
        };
        double2 a0 = make_double2(0.0, 0.0);
#pragma unroll
        for (int p = 1; p < NPC; ++p) {
          const double2 d = live ? cscale(csub(pa, R[j4_at(B, s2, c, p)]), wt[c * NPC + p]) : make_double2(0.0, 0.0);
          a0 = cadd(a0, d);
          put(p, make_double2(-d.x, -d.y));
        }
        {  // storativity block: K = s2 2 + comp in step KS
          const double2 As = live ? cmul(wz[k], cscale(pa, wt[c * NPC])) : make_double2(0.0, 0.0);
          Ac[KS * 32 + lrow + s2 * 2] = As.x;
          Ac[KS * 32 + lrow + s2 * 2 + 1] = -As.y;
        }
      }
      __syncwarp();
      if (lane == 0) {
        jw_arrive(&a_full[t % J4_NA]);
        jw_arrive(&raw_empty[t % J4_NRAW]);
      }
    }
  } else {
    // ------------------------------- consumers -------------------------------------------
    const int kq = lane & 3, rl = lane >> 2;
    const int rcol = n_src + min(wc * 8 + rl, n_rec - 1);
    // lane-constant B-operand offsets (doubles from the slot base) of every K step, cell 0;
    // cell c adds c B complex in every region.  Step KS is the storativity block (centre point).
    int offk[KS + 1];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int K = ks * 4 + kq, s2 = K / (2 * NF), p = 1 + (K >> 1) % NF;
      offk[ks] = 2 * j4_at(B, s2, 0, p) + 2 * rcol + (K & 1);
    }
    const int offc0 = 2 * j4_at(B, 0, 0, 0) + 2 * rcol + (kq & 1), offc1 = 2 * j4_at(B, 1, 0, 0) + 2 * rcol + (kq & 1);
    offk[KS] = 2 * j4_at(B, kq >> 1, 0, 0) + 2 * rcol + (kq & 1);
    const int cstep = 2 * B;
    double accK[J4_TC][2][2], accS[J4_TC][2][2];  // [cell][m tile][2]
    for (int t = 0; t < T; ++t) {
      if (t % npair == 0) {
#pragma unroll
        for (int c = 0; c < J4_TC; ++c)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) accK[c][mt][0] = accK[c][mt][1] = accS[c][mt][0] = accS[c][mt][1] = 0.0;
      }
      jw_wait(&raw_full[t % J4_NRAW], (uint32_t)((t / J4_NRAW) & 1));
      jw_wait(&a_full[t % J4_NA], (uint32_t)((t / J4_NA) & 1));
      const double* rw = reinterpret_cast<const double*>(raw + (t % J4_NRAW) * SLOT);
      const double* Al = Af + (t % J4_NA) * AF + lane;
      // K steps outer, cells inner: 8 independent accumulator chains per step
#pragma unroll
      for (int ks = 0; ks <= KS; ++ks) {
        double bv[J4_TC], a0[J4_TC], a1[J4_TC];
#pragma unroll
        for (int c = 0; c < J4_TC; ++c) {
          bv[c] = rw[offk[ks] + c * cstep];
          if (ks < KS) bv[c] -= rw[((ks * 4) / (2 * NF) == 0 ? offc0 : offc1) + c * cstep];
          a0[c] = Al[c * 2 * MTS + ks * 32];
          a1[c] = Al[c * 2 * MTS + MTS + ks * 32];
        }
#pragma unroll
        for (int c = 0; c < J4_TC; ++c) {
          if (ks < KS) {
            dmma(accK[c][0], a0[c], bv[c]);
            dmma(accK[c][1], a1[c], bv[c]);
          } else {
            dmma(accS[c][0], a0[c], bv[c]);
            dmma(accS[c][1], a1[c], bv[c]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        jw_arrive(&a_empty[t % J4_NA]);
        jw_arrive(&raw_empty[t % J4_NRAW]);
      }
      if (t % npair == npair - 1) {
        const TileXY g = tile_at(t);
        const int64_t a = ((int64_t)g.kz * L.ny + g.j) * L.nx + g.i0;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int s = mt * 8 + (lane >> 2);
          if (s >= n_src) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wc * 8 + (lane & 3) * 2 + h;
            if (r >= n_rec) continue;
            const int64_t o = ((int64_t)s * n_rec + r) * ldj + a;
            stg256(Jk + o, 2.0 * accK[0][mt][h], 2.0 * accK[1][mt][h], 2.0 * accK[2][mt][h], 2.0 * accK[3][mt][h], pol);
            if (Js)
              stg256(Js + o, 2.0 * accS[0][mt][h], 2.0 * accS[1][mt][h], 2.0 * accS[2][mt][h], 2.0 * accS[3][mt][h],
                     pol);
          }
        }
      }
    }
  }
}

// P1 rows (sensitivity_row_conductivity / _storativity, jacobian.cpp:57-125) on the node
// grid of build_mesh: per element e (2c lower (a,b,c), 2c+1 upper (a,c,d) of cell c)
//   J_k[e] = 2 Re sum_k w_k (kappa_e / 2) (D0 phi D0 psi + D1 phi D1 psi)
//     (exact P1 gradients: area h^2/2, grad = edge differences / h)
//   J_S[e] = 2 Re sum_k w_k z_k (S_e h^2 / 24) ((sum phi)(sum psi) + sum_i phi_i psi_i)
//     (exact P1 product integral area/12 sum (1 + d_ij) phi_i psi_j)
// Dirichlet nodes carry zero.  A CTA owns TC cells (2 TC elements) of one row.
__global__ void __launch_bounds__(kT, 2) jacobian_p1_kernel(int nx, double h2, const double* __restrict__ kappa,
                                                            const double* __restrict__ stor,
                                                            const double2* __restrict__ fields, int n_src, int n_rec,
                                                            int ns, const double2* __restrict__ w,
                                                            const double2* __restrict__ wz, int TC, int tiles_x,
                                                            int nsub_r, int nsub_total, double* __restrict__ Jk,
                                                            double* __restrict__ Js, int64_t ldj) {
  extern __shared__ double2 smem[];
  const int n_items = n_src + n_rec;
  const int U = 2 * TC;                                  // elements per tile
  double2* P = smem;                                     // [4][n_src][U]
  double2* Q = smem + (size_t)4 * n_src * U;             // [4][n_rec][U]
  double* wt = reinterpret_cast<double*>(Q + (size_t)4 * n_rec * U);  // [2][U]: kappa_e/2, S_e h^2/24
  const int nc = nx + 1;
  const int64_t n = (int64_t)nx * nx;
  const int cj = blockIdx.x / tiles_x;
  const int ci0 = (blockIdx.x % tiles_x) * TC;
  const int ncell = min(TC, nc - ci0);
  const int tid = threadIdx.x;
  const int c = tid % U;
  const int sub = tid / U;
  const bool owner = sub < nsub_total && (c >> 1) < ncell;
  const int s0 = owner ? (sub / nsub_r) * SB : 0;
  const int r0 = owner ? (sub % nsub_r) * RB : 0;
  if (tid < U) {
    const int ci = ci0 + (tid >> 1);
    const int64_t e = 2 * ((int64_t)cj * nc + ci) + (tid & 1);
    wt[tid] = (tid >> 1) < ncell ? 0.5 * kappa[e] : 0.0;
    wt[U + tid] = (tid >> 1) < ncell ? stor[e] * h2 / 24.0 : 0.0;
  }
  __syncthreads();
  auto nodev = [&](const double2* fld, int I, int J) {
    return (I >= 1 && I <= nx && J >= 1 && J <= nx) ? fld[(int64_t)(J - 1) * nx + (I - 1)] : make_double2(0.0, 0.0);
  };
  for (int phase = 0; phase < (Js ? 2 : 1); ++phase) {
    const int nstage = phase == 0 ? 2 : 4;
    double acc[SB][RB];
#pragma unroll
    for (int i = 0; i < SB; ++i)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[i][q] = 0.0;
    for (int k = 0; k < ns; ++k) {
      const double2 wk = phase == 0 ? w[k] : wz[k];
      for (int e = tid; e < n_items * TC; e += blockDim.x) {
        const int it = e / TC, cc = e % TC;
        double2 v[2][4];
        if (cc < ncell) {
          const double2* fld = fields + ((int64_t)it * ns + k) * n;
          const int ci = ci0 + cc;
          const double2 fa = nodev(fld, ci, cj), fb = nodev(fld, ci + 1, cj);
          const double2 fc = nodev(fld, ci + 1, cj + 1), fd = nodev(fld, ci, cj + 1);
          if (phase == 0) {
            v[0][0] = csub(fb, fa); v[0][1] = csub(fc, fb);  // lower (a, b, c)
            v[1][0] = csub(fc, fd); v[1][1] = csub(fd, fa);  // upper (a, c, d)
          } else {
            v[0][0] = cadd(cadd(fa, fb), fc); v[0][1] = fa; v[0][2] = fb; v[0][3] = fc;
            v[1][0] = cadd(cadd(fa, fc), fd); v[1][1] = fa; v[1][2] = fc; v[1][3] = fd;
          }
        } else {
          for (int q = 0; q < 4; ++q) v[0][q] = v[1][q] = make_double2(0.0, 0.0);
        }
        for (int el = 0; el < 2; ++el) {
          const int u = 2 * cc + el;
          for (int f = 0; f < nstage; ++f) {
            if (it < n_src) P[((size_t)f * n_src + it) * U + u] = cscale(cmul(wk, v[el][f]), wt[phase * U + u]);
            else Q[((size_t)f * n_rec + (it - n_src)) * U + u] = v[el][f];
          }
        }
      }
      __syncthreads();
      if (owner) {
#pragma unroll 1
        for (int f = 0; f < nstage; ++f) {
          double2 pv[SB];
#pragma unroll
          for (int i = 0; i < SB; ++i)
            pv[i] = (s0 + i < n_src) ? P[((size_t)f * n_src + s0 + i) * U + c] : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const double2 qv = (r0 + q < n_rec) ? Q[((size_t)f * n_rec + r0 + q) * U + c] : make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < SB; ++i) acc[i][q] = fma(pv[i].x, qv.x, fma(-pv[i].y, qv.y, acc[i][q]));
          }
        }
      }
      __syncthreads();
    }
    if (owner) {
      double* Jout = phase == 0 ? Jk : Js;
      const int64_t e = 2 * ((int64_t)cj * nc + ci0 + (c >> 1)) + (c & 1);
#pragma unroll
      for (int i = 0; i < SB; ++i) {
        if (s0 + i >= n_src) continue;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          if (r0 + q >= n_rec) continue;
          Jout[((int64_t)(s0 + i) * n_rec + (r0 + q)) * ldj + e] = 2.0 * acc[i][q];
        }
      }
    }
  }
}

struct PointSet {
  std::vector<int64_t> idx;  // n_pts * 8
  std::vector<double> w;
  std::vector<int> cnt;
};

PointSet make_points(lt_pencil p, const double* pts, int n_pts) {
  PointSet ps;
  ps.idx.assign((size_t)n_pts * 8, 0);
  ps.w.assign((size_t)n_pts * 8, 0.0);
  ps.cnt.assign(n_pts, 0);
  for (int r = 0; r < n_pts; ++r)
    point_weights(p, pts + (size_t)r * p->dim, ps.idx.data() + r * 8, ps.w.data() + r * 8, &ps.cnt[r]);
  return ps;
}

void throw_unconverged(const OuterResult& res, const char* what) {
  for (int b = 0; b < res.B; ++b) {
    std::vector<int> bad;
    for (int k = 0; k < res.n_shifts; ++k)
      if (!res.status[(size_t)b * res.n_shifts + k].converged) bad.push_back(k);
    if (!bad.empty()) {
      g_last_unconverged = bad;
      throw Error(LT_ERR_NOT_CONVERGED, std::string(what) + ": " + std::to_string(bad.size()) + " of " +
                                            std::to_string(res.n_shifts) + " shifts unconverged after " +
                                            std::to_string(res.iterations[b]) + " iterations");
    }
  }
}

// Shifts and schedule of one family (solve_family, forward.cpp:40-71).
void fill_schedule(OuterProblem& prob, int b, const std::vector<cd>& shifts, int kind, int maxit_eff) {
  Schedule sch = select_schedule(shifts);
  if (kind == LT_SOLVER_SINGLE) {
    sch.taus = {sch.taus[0]};
    sch.pattern = {0};
  }
  prob.tau_table[b].resize(maxit_eff);
  for (int j = 0; j < maxit_eff; ++j) prob.tau_table[b][j] = d2(sch.tau_at(j));
  for (size_t k = 0; k < shifts.size(); ++k) prob.shifts[(size_t)b * shifts.size() + k] = d2(shifts[k]);
}

int effective_maxit(int64_t n, int maxit, int ns) {
  return maxit > 0 ? (int)std::min<int64_t>(n, maxit) : (int)std::min<int64_t>(n, 10 * (int64_t)ns);
}

// Direct mode (solve_shifted_direct, cpp:324-332): one shift-and-invert solve per shift, stored
// as a basis whose coefficient vectors select column k.  The reference's LU is exact; here each
// solve's final relative residual is reported as the shift's true residual, and a shift whose
// solve ended above `tol` is unconverged (the driver then raises ConvergenceError).
void direct_solve(lt_pencil p, int B, const double2* b_dev, const std::vector<cd>& shifts_all, int ns, double tol,
                  OuterResult& res) {
  cudaStream_t st = p->ctx->stream;
  const int64_t n = p->n;
  res.B = B;
  res.n_shifts = ns;
  res.maxit = ns;
  res.cap = ns;
  res.iterations.assign(B, 0);
  res.status.assign((size_t)B * ns, lt_shift_status{1, 1, 0.0, 0.0});
  res.m_used.assign((size_t)B * ns, 0);
  res.U.clear();
  std::vector<double2> Y((size_t)B * ns * ns, make_double2(0, 0));
  for (int k = 0; k < ns; ++k) {
    res.U.emplace_back(sizeof(double2) * (size_t)B * n, st);
    std::vector<double2> taus(B);
    for (int b = 0; b < B; ++b) taus[b] = d2(shifts_all[(size_t)b * ns + k]);
    std::vector<double> rel(B, 0.0);
    inner_solve(p, B, taus.data(), b_dev, n, res.U.back().as<double2>(), n, nullptr, rel.data());
    for (int b = 0; b < B; ++b) {
      res.status[(size_t)b * ns + k] = lt_shift_status{rel[b] <= tol, 1, rel[b], rel[b]};
      Y[((size_t)b * ns + k) * ns + k] = make_double2(1.0, 0.0);
      res.m_used[(size_t)b * ns + k] = k + 1;
    }
  }
  res.Y.allocate(sizeof(double2) * Y.size(), st);
  LT_CUDA(cudaMemcpyAsync(res.Y.get(), Y.data(), sizeof(double2) * Y.size(), cudaMemcpyHostToDevice, st));
}

// Run one batch of families (same n_shifts) with the configured solver.
void solve_families(lt_pencil p, const lt_solver_config& cfg, int B, const double2* b_dev,
                    const std::vector<std::vector<cd>>& shifts, OuterResult& res) {
  const int ns = (int)shifts[0].size();
  if (cfg.kind == LT_SOLVER_DIRECT) {
    std::vector<cd> all;
    for (auto& s : shifts) all.insert(all.end(), s.begin(), s.end());
    direct_solve(p, B, b_dev, all, ns, cfg.tol, res);
    return;
  }
  OuterProblem prob;
  prob.B = B;
  prob.n_shifts = ns;
  prob.b = b_dev;
  prob.variant = cfg.variant;
  prob.tol = cfg.tol;
  prob.maxit = cfg.maxit;
  prob.record_history = false;
  const int me = effective_maxit(p->n, cfg.maxit, ns);
  prob.shifts.resize((size_t)B * ns);
  prob.tau_table.resize(B);
  for (int b = 0; b < B; ++b) fill_schedule(prob, b, shifts[b], cfg.kind, me);
  outer_solve(p, prob, res);
}

// c[b][j] = sum_k coef[b][k] y[b][k][j]  (j < m_used[b][k])
std::vector<double2> basis_coefficients(const OuterResult& res, const std::vector<cd>& coef, int& mc,
                                        int k_begin, int k_end, cudaStream_t st) {
  const int B = res.B, ns = res.n_shifts;
  std::vector<double2> Y((size_t)B * ns * res.maxit);
  LT_CUDA(cudaMemcpyAsync(Y.data(), res.Y.get(), sizeof(double2) * Y.size(), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  mc = (int)res.U.size();
  std::vector<double2> c((size_t)B * std::max(mc, 1), make_double2(0, 0));
  for (int b = 0; b < B; ++b)
    for (int k = k_begin; k < k_end; ++k) {
      const cd ck = coef[(size_t)b * ns + k];
      const int mu = res.m_used[(size_t)b * ns + k];
      for (int j = 0; j < mu; ++j) {
        const double2 y = Y[((size_t)b * ns + k) * res.maxit + j];
        const cd v = ck * cd(y.x, y.y);
        c[(size_t)b * mc + j].x += v.real();
        c[(size_t)b * mc + j].y += v.imag();
      }
    }
  return c;
}

void recombine(lt_pencil p, const OuterResult& res, const std::vector<double2>& c, int mc,
               const std::vector<int64_t>& dst, double* heads_dev) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  const int B = res.B;
  std::vector<const double2*> cols(std::max(mc, 1), nullptr);
  for (int j = 0; j < mc; ++j) cols[j] = res.U[j].as<double2>();
  DeviceBuffer dcols(sizeof(void*) * cols.size(), st), dc(sizeof(double2) * c.size(), st),
      ddst(sizeof(int64_t) * dst.size(), st);
  LT_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(void*) * cols.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dc.get(), c.data(), sizeof(double2) * c.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(ddst.get(), dst.data(), sizeof(int64_t) * dst.size(), cudaMemcpyHostToDevice, st));
  launch(ctx, "recombine", (double)n * B * (16.0 * mc + 16.0), [&] {
    recombine_kernel<<<blocks_for(n, kT) * B, kT, 0, st>>>(n, B, mc, dcols.as<const double2*>(), dc.as<double2>(),
                                                            ddst.as<int64_t>(), heads_dev);
  });
  stream_sync(ctx);
}

}  // namespace

void forward(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
             const double* times, int n_times, int n_quad, const lt_talbot_params& contour, const lt_solver_config& cfg,
             bool pooled, int mem, double* heads_out, const double* receivers, int n_rec, double* drawdown_out,
             lt_time_diag* diag_out, double* shift_residuals) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  LT_REQUIRE(n_src >= 1, "solve_forward: no source");
  LT_REQUIRE(n_times >= 1, "solve_forward: no target times");
  double previous = 0.0;
  for (int t = 0; t < n_times; ++t) {
    LT_REQUIRE(times[t] > 0.0, "solve_forward: times must be positive");
    LT_REQUIRE(times[t] >= previous, "solve_forward: times must be ascending");
    previous = times[t];
  }
  LT_REQUIRE(n_quad >= 4 && n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
  const int nh = n_quad / 2;
  std::vector<std::vector<cd>> nodes(n_times), weights(n_times);
  for (int t = 0; t < n_times; ++t) talbot_build(n_quad, times[t], contour, nullptr, &nodes[t], nullptr, &weights[t]);

  // host copies of the source vectors (and initial heads) for the families
  auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DeviceBuffer src_dev(sizeof(double) * (size_t)n * n_src, st);
  LT_CUDA(cudaMemcpyAsync(src_dev.get(), sources, sizeof(double) * n * n_src, kind, st));
  std::vector<double> ih_h;
  std::vector<int> with_initial(n_src, 0);
  DeviceBuffer ih_dev;
  if (initial_head) {
    ih_dev.allocate(sizeof(double) * (size_t)n * n_src, st);
    LT_CUDA(cudaMemcpyAsync(ih_dev.get(), initial_head, sizeof(double) * n * n_src, kind, st));
    ih_h.resize((size_t)n * n_src);
    LT_CUDA(cudaMemcpyAsync(ih_h.data(), ih_dev.get(), sizeof(double) * n * n_src, cudaMemcpyDeviceToHost, st));
  }
  stream_sync(ctx);
  for (int s = 0; s < n_src && initial_head; ++s) {
    double mx = 0.0;
    for (int64_t a = 0; a < n; ++a) mx = std::max(mx, std::fabs(ih_h[(size_t)s * n + a]));
    with_initial[s] = mx > 0.0;
  }

  // Families: (source, time) items with the rate transform, and (source, time) items with
  // rhs M phi0 when the initial head is nonzero.  Pooled mode: one item per source with the
  // pooled shifts of every time.
  struct Fam { int s; int t; bool initial; };
  std::vector<Fam> fams;
  for (int s = 0; s < n_src; ++s) {
    if (pooled) {
      if (rates[s] != 0.0) fams.push_back({s, -1, false});
      if (with_initial[s]) fams.push_back({s, -1, true});
    } else {
      for (int t = 0; t < n_times; ++t) {
        if (rates[s] != 0.0) fams.push_back({s, t, false});
        if (with_initial[s]) fams.push_back({s, t, true});
      }
    }
  }
  const int F = (int)fams.size();
  const int ns = pooled ? nh * n_times : nh;
  DeviceBuffer heads_dev(sizeof(double) * (size_t)n * n_times * n_src, st);
  LT_CUDA(cudaMemsetAsync(heads_dev.get(), 0, heads_dev.bytes(), st));
  std::vector<lt_time_diag> diags(n_times, lt_time_diag{0, 1});
  if (shift_residuals)
    for (size_t q = 0; q < (size_t)n_src * n_times * nh; ++q) shift_residuals[q] = NAN;

  // item chunks bounded by memory: ~ (2 maxit-columns) vectors per item
  const double per_item = (double)n * sizeof(double2) * 14.0;
  const int chunk = std::max(1, (int)std::min<double>(F, 0.6 * available_device_bytes(p->ctx) / per_item));

  for (int f0 = 0; f0 < F; f0 += chunk) {
    const int B = std::min(chunk, F - f0);
    // right-hand sides
    DeviceBuffer rhs(sizeof(double2) * (size_t)B * n, st);
    std::vector<std::vector<cd>> shifts(B);
    for (int q = 0; q < B; ++q) {
      const Fam& fm = fams[f0 + q];
      if (pooled) {
        for (int t = 0; t < n_times; ++t) shifts[q].insert(shifts[q].end(), nodes[t].begin(), nodes[t].end());
      } else {
        shifts[q] = nodes[fm.t];
      }
      double2* dst = rhs.as<double2>() + (size_t)q * n;
      if (!fm.initial) {
        const double* srcp = src_dev.as<double>() + (size_t)fm.s * n;
        launch(ctx, "rhs", 24.0 * n, [&] { real_to_complex<<<blocks_for(n, kT), kT, 0, st>>>(n, srcp, dst); });
      } else {
        // rhs = M phi0 (apply_mass, forward.cpp:91-93)
        DeviceBuffer tmp(sizeof(double2) * n, st);
        const double* ihp = ih_dev.as<double>() + (size_t)fm.s * n;
        launch(ctx, "rhs", 24.0 * n, [&] { real_to_complex<<<blocks_for(n, kT), kT, 0, st>>>(n, ihp, tmp.as<double2>()); });
        apply_batch(p, 0, nullptr, tmp.as<double2>(), n, dst, n, 1, true, "apply_mass");
      }
    }
    OuterResult res;
    solve_families(p, cfg, B, rhs.as<double2>(), shifts, res);
    // diagnostics and convergence (forward.cpp:57-69)
    for (int q = 0; q < B; ++q) {
      const Fam& fm = fams[f0 + q];
      for (int t = 0; t < n_times; ++t) {
        if (!pooled && fm.t != t) continue;
        diags[t].iterations = std::max(diags[t].iterations, res.iterations[q]);
        for (int k = 0; k < ns; ++k) {
          const auto& stt = res.status[(size_t)q * ns + k];
          if (!stt.converged) diags[t].all_converged = 0;
        }
      }
      if (shift_residuals && !fm.initial) {
        for (int k = 0; k < ns; ++k) {
          const int t = pooled ? k / nh : fm.t;
          const int kk = pooled ? k % nh : k;
          shift_residuals[((size_t)fm.s * n_times + t) * nh + kk] = res.status[(size_t)q * ns + k].true_residual;
        }
      }
    }
    throw_unconverged(res, pooled ? "batch solve" : "shifted solve");
    // recombination per time into heads[s][t]
    for (int t = 0; t < n_times; ++t) {
      std::vector<cd> coef((size_t)B * ns, cd(0.0, 0.0));
      bool any = false;
      for (int q = 0; q < B; ++q) {
        const Fam& fm = fams[f0 + q];
        if (!pooled && fm.t != t) continue;
        any = true;
        for (int k = 0; k < nh; ++k) {
          const int kk = pooled ? t * nh + k : k;
          const cd z = nodes[t][k];
          const cd qh = fm.initial ? cd(1.0, 0.0) : rates[fm.s] / z;  // qhat_step
          coef[(size_t)q * ns + kk] = weights[t][k] * qh;
        }
      }
      if (!any) continue;
      int mc = 0;
      std::vector<double2> c = basis_coefficients(res, coef, mc, 0, ns, st);
      // two passes so the rate and initial-head families of one (s, t) never race
      for (int pass = 0; pass < 2; ++pass) {
        std::vector<int64_t> dst(B, -1);
        bool anyp = false;
        for (int q = 0; q < B; ++q) {
          const Fam& fm = fams[f0 + q];
          if ((!pooled && fm.t != t) || (int)fm.initial != pass) continue;
          dst[q] = ((int64_t)fm.s * n_times + t) * n;
          anyp = true;
        }
        if (anyp) recombine(p, res, c, mc, dst, heads_dev.as<double>());
      }
      stream_sync(ctx);
    }
  }
  if (heads_out) {
    auto k2 = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    LT_CUDA(cudaMemcpyAsync(heads_out, heads_dev.get(), sizeof(double) * (size_t)n * n_times * n_src, k2, st));
  }
  if (receivers && n_rec > 0 && drawdown_out) {
    PointSet ps = make_points(p, receivers, n_rec);
    DeviceBuffer didx(sizeof(int64_t) * ps.idx.size(), st), dw(sizeof(double) * ps.w.size(), st),
        dcnt(sizeof(int) * ps.cnt.size(), st), dout(sizeof(double) * (size_t)n_src * n_times * n_rec, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), ps.idx.data(), sizeof(int64_t) * ps.idx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dw.get(), ps.w.data(), sizeof(double) * ps.w.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), ps.cnt.data(), sizeof(int) * ps.cnt.size(), cudaMemcpyHostToDevice, st));
    const int Bh = n_src * n_times;
    launch(ctx, "gather_points", 0.0, [&] {
      gather_points<<<blocks_for((int64_t)Bh * n_rec, 128), 128, 0, st>>>(n, Bh, n_rec, heads_dev.as<double>(),
                                                                          didx.as<int64_t>(), dw.as<double>(), dcnt.as<int>(),
                                                                          dout.as<double>());
    });
    std::vector<double> g((size_t)Bh * n_rec);
    LT_CUDA(cudaMemcpyAsync(g.data(), dout.get(), sizeof(double) * g.size(), cudaMemcpyDeviceToHost, st));
    stream_sync(ctx);
    // reorder (s, t, r) -> (s, r, t)  (ThtExperiment::measurement_index, jacobian.hpp:37-41)
    for (int s = 0; s < n_src; ++s)
      for (int t = 0; t < n_times; ++t)
        for (int r = 0; r < n_rec; ++r)
          drawdown_out[((size_t)s * n_rec + r) * n_times + t] = g[((size_t)s * n_times + t) * n_rec + r];
  }
  stream_sync(ctx);
  if (diag_out)
    for (int t = 0; t < n_times; ++t) diag_out[t] = diags[t];
}

// FD with <= 16 sources and <= 64 receivers: the tensor-core Jacobian on cell-major fields
bool use_tensor_jacobian(lt_pencil p, int n_src, int n_rec) {
  const int B = n_src + n_rec;
  return p->kind != LT_GRID_P1_TRI && n_src <= JW_SMAX && n_rec <= JW_RMAX && 2 * B <= 256 &&
         (p->dim == 3 ? jw_smem<3>(B) : jw_smem<2>(B)) <= 227 * 1024;
}

// The forward (sources, b_s) and adjoint (receivers, -e_r) shifted families of items
// [item0, item1) of one time slice (jacobian.cpp:205-227; items = sources then receivers) as one
// lockstep FGMRES-Sh batch; raises ConvergenceError like solve_family_or_throw (cpp:19-43).
void solve_slice_items(lt_pencil p, const lt_experiment& ex, const std::vector<cd>& nodes, int item0, int item1,
                       OuterResult& res) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int n_src = ex.n_src, n_rec = ex.n_rec, ns = ex.n_quad / 2;
  const int64_t n = p->n;
  PointSet src = make_points(p, ex.sources, n_src);
  PointSet rec = make_points(p, ex.receivers, n_rec);
  const int BT = n_src + n_rec;
  LT_REQUIRE(item0 >= 0 && item0 < item1 && item1 <= BT, "jacobian: bad item range");
  // rhs: sources b_s, receivers -e_r  (jacobian.cpp:216, 227, solve_adjoint_fields cpp:49)
  // sparse point weights of all items (sources +w, receivers -w), scattered on the device
  std::vector<int64_t> pidx((size_t)BT * 8, 0);
  std::vector<double> pw((size_t)BT * 8, 0.0);
  std::vector<int> pcnt(BT, 0);
  for (int s = 0; s < n_src; ++s) {
    pcnt[s] = src.cnt[s];
    for (int q = 0; q < src.cnt[s]; ++q) { pidx[s * 8 + q] = src.idx[s * 8 + q]; pw[s * 8 + q] = src.w[s * 8 + q]; }
  }
  for (int r = 0; r < n_rec; ++r) {
    pcnt[n_src + r] = rec.cnt[r];
    for (int q = 0; q < rec.cnt[r]; ++q) {
      pidx[(n_src + r) * 8 + q] = rec.idx[r * 8 + q];
      pw[(n_src + r) * 8 + q] = -rec.w[r * 8 + q];
    }
  }
  // this part's items only
  const int B = item1 - item0;
  pidx.erase(pidx.begin(), pidx.begin() + (size_t)item0 * 8);
  pw.erase(pw.begin(), pw.begin() + (size_t)item0 * 8);
  pcnt.erase(pcnt.begin(), pcnt.begin() + item0);
  DeviceBuffer rhs(sizeof(double2) * (size_t)B * n, st);
  {
    DeviceBuffer didx(sizeof(int64_t) * pidx.size(), st), dwt(sizeof(double) * pw.size(), st), dcnt(sizeof(int) * B, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), pidx.data(), sizeof(int64_t) * pidx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dwt.get(), pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), pcnt.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemsetAsync(rhs.get(), 0, rhs.bytes(), st));
    launch(ctx, "rhs", 0.0, [&] {
      scatter_points<<<blocks_for((int64_t)B * 8, 128), 128, 0, st>>>(n, B, didx.as<int64_t>(), dwt.as<double>(),
                                                                      dcnt.as<int>(), rhs.as<double2>());
    });
  }
  std::vector<std::vector<cd>> shifts(B, nodes);
  {
    TraceScope tr(ctx, "  solve_families", B);
    solve_families(p, ex.solver, B, rhs.as<double2>(), shifts, res);
  }
  // forward failures first (jacobian.cpp:214-218), then adjoint
  {
    OuterResult* r = &res;
    for (int b = 0; b < B; ++b) {
      std::vector<int> bad;
      for (int k = 0; k < ns; ++k)
        if (!r->status[(size_t)b * ns + k].converged) bad.push_back(k);
      if (!bad.empty()) {
        g_last_unconverged = bad;
        throw Error(LT_ERR_NOT_CONVERGED, std::string(item0 + b < n_src ? "forward solve" : "adjoint solve") + ": " +
                                              std::to_string(bad.size()) + " of " + std::to_string(ns) +
                                              " shifts unconverged after " + std::to_string(r->iterations[b]) + " iterations");
      }
    }
  }
}

// FD Jacobian rows of every (source, receiver) pair over the cells of the view Lv (the whole
// fine grid, or a z-slab with its halo planes for the split build): J[(s n_rec + r) ldj + a]
// (kappa block) and J[... + s_off + a] (storativity block, include_s), fields over the view's
// cells, cell-major for the tensor-core kernels (tensor_jac) else RHS-major; dw = the w_k then
// wz_k factors (n_shifts each).  kappa / stor are the view's per-cell fields.
void fd_jacobian_kernels(lt_pencil p, const LevelView& Lv, const double* kappa, const double* stor,
                         const double2* fields, int n_src, int n_rec, int ns, const double2* dw, bool tensor_jac,
                         bool include_s, double* J, int64_t ldj, int64_t s_off) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int B = n_src + n_rec;
  const double h = p->grid.h;
  const double face_scale = p->dim == 3 ? h : 1.0;
  const double hd = p->dim == 3 ? h * h * h : h * h;
  const double bytes = (double)Lv.n * (16.0 * ns * B + 8.0 * n_src * n_rec * (include_s ? 2 : 1));
  // 4-cell tiles with 32-byte J stores where rows allow it (2-cell tiles otherwise)
  const bool tile4 = tensor_jac && Lv.nx % J4_TC == 0 && ldj % 4 == 0 && s_off % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(J) & 31) == 0 &&
                     (p->dim == 3 ? j4_smem<3>(B) : j4_smem<2>(B)) <= 227 * 1024;
  if (tile4) {
    const LevelView& L = Lv;
    const int ntiles = (L.nx / J4_TC) * L.ny * L.nz;
    const int grid = std::min(ntiles, ctx->num_sms);
    const size_t smem = p->dim == 3 ? j4_smem<3>(B) : j4_smem<2>(B);
    auto fn = p->dim == 3 ? jacobian_mma4_kernel<3> : jacobian_mma4_kernel<2>;
    LT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint64_t dims[5] = {2 * (uint64_t)B, (uint64_t)L.nx, (uint64_t)L.ny, (uint64_t)L.nz, (uint64_t)ns};
    const uint64_t strd[4] = {(uint64_t)B * 16, (uint64_t)L.nx * B * 16, (uint64_t)L.nx * L.ny * B * 16,
                              (uint64_t)Lv.n * B * 16};
    const uint32_t boxC[5] = {2 * (uint32_t)B, 6, 1, 1, 2}, boxF[5] = {2 * (uint32_t)B, 4, 1, 1, 2};
    const CUtensorMap mC = tma_map_8b((void*)fields, 5, dims, strd, boxC);
    const CUtensorMap mF = tma_map_8b((void*)fields, 5, dims, strd, boxF);
    launch(ctx, "jacobian", bytes, [&] {
      fn<<<grid, J4_THREADS, smem, st>>>(mC, mF, L, kappa, stor, hd,
                                         face_scale, n_src, n_rec, ns, dw + ns, J,
                                         include_s ? J + s_off : nullptr, ldj, ntiles);
    });
  } else if (tensor_jac) {
    const LevelView& L = Lv;
    const int ntiles = ((L.nx + JW_TC - 1) / JW_TC) * L.ny * L.nz;
    const int grid = std::min(ntiles, ctx->num_sms);
    const size_t smem = p->dim == 3 ? jw_smem<3>(B) : jw_smem<2>(B);
    auto fn = p->dim == 3 ? jacobian_mma_kernel<3> : jacobian_mma_kernel<2>;
    LT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // 5-D maps over the cell-major fields: (item re/im, x, y, z, shift)
    const uint64_t dims[5] = {2 * (uint64_t)B, (uint64_t)L.nx, (uint64_t)L.ny, (uint64_t)L.nz, (uint64_t)ns};
    const uint64_t strd[4] = {(uint64_t)B * 16, (uint64_t)L.nx * B * 16, (uint64_t)L.nx * L.ny * B * 16,
                              (uint64_t)Lv.n * B * 16};
    const uint32_t boxA[5] = {2 * (uint32_t)B, 4, 3, 1, 2}, boxB[5] = {2 * (uint32_t)B, 2, 1, 3, 2};
    const CUtensorMap mA = tma_map_8b((void*)fields, 5, dims, strd, boxA);
    const CUtensorMap mB = tma_map_8b((void*)fields, 5, dims, strd, boxB);
    launch(ctx, "jacobian", bytes, [&] {
      fn<<<grid, JW_THREADS, smem, st>>>(mA, mB, L, kappa, stor, hd,
                                         face_scale, n_src, n_rec, ns, nullptr, dw + ns, J,
                                         include_s ? J + s_off : nullptr, ldj, ntiles);
    });
  } else {
    const int nsub_s = (n_src + SB - 1) / SB, nsub_r = (n_rec + RB - 1) / RB;
  const int nsub_total = nsub_s * nsub_r;
  LT_REQUIRE(nsub_total <= kT, "jacobian: too many source/receiver blocks for one CTA (n_src*n_rec too large)");
  const int nf = 2 * p->dim + 1;
  int TC = std::max(1, kT / nsub_total);
  const LevelView& L = Lv;
  TC = std::min(TC, L.nx);
  auto smem_for = [&](int tc) {
    return sizeof(double2) * (size_t)(nf - 1) * B * tc + sizeof(double) * nf * tc + sizeof(int64_t) * 2 * p->dim * tc;
  };
  while (TC > 1 && smem_for(TC) > 110 * 1024) TC /= 2;  // two CTAs per SM
  LT_REQUIRE(nf * TC <= kT, "jacobian: tile too wide");
  const size_t smem = smem_for(TC);
  const int tiles_x = (L.nx + TC - 1) / TC;
  const unsigned grid = (unsigned)(tiles_x * (int64_t)L.ny * L.nz);
  auto fn = p->dim == 3 ? jacobian_kernel<3> : jacobian_kernel<2>;
  LT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  launch(ctx, "jacobian", bytes, [&] {
    fn<<<grid, kT, smem, st>>>(L, kappa, stor, hd, face_scale,
                               fields, n_src, n_rec, ns, dw, dw + ns, TC,
                               tiles_x, nsub_r, nsub_total, J, include_s ? J + s_off : nullptr, ldj);
  });
  }
}

void jacobian_slice(lt_pencil p, const lt_experiment& ex, int t, int mem, double* jac_out, double* pred_out) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  const int n_src = ex.n_src, n_rec = ex.n_rec;
  LT_REQUIRE(n_src >= 1 && n_rec >= 1 && ex.n_times >= 1, "ThtForwardModel: experiment must be nonempty");
  LT_REQUIRE(t >= 0 && t < ex.n_times, "jacobian_slice: time index out of range");
  LT_REQUIRE(!(jac_out && p->from_csr),
             "ThtForwardModel::jacobian: the pencil was created from (K, M) and carries no parameter fields");
  LT_REQUIRE(ex.n_quad >= 4 && ex.n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
  LT_REQUIRE(ex.times[t] > 0.0, "build_contour: time must be positive");
  TraceScope trace_all(ctx, "jacobian_slice", t);
  const int ns = ex.n_quad / 2;
  std::vector<cd> nodes, weights;
  talbot_build(ex.n_quad, ex.times[t], ex.contour, nullptr, &nodes, nullptr, &weights);

  const int B = n_src + n_rec;
  OuterResult res;
  solve_slice_items(p, ex, nodes, 0, B, res);
  const PointSet rec = make_points(p, ex.receivers, n_rec);
  // fields: phi_{s,k} = qhat_k U_s y_{s,k}; psi_{r,k} = U_r y_{r,k}
  std::vector<double2> scale((size_t)B * ns, make_double2(1.0, 0.0));
  for (int s = 0; s < n_src; ++s)
    for (int k = 0; k < ns; ++k) scale[(size_t)s * ns + k] = d2(ex.rates[s] / nodes[k]);
  // FD with <= 16 sources and <= 64 receivers: tensor-core Jacobian on cell-major fields (the
  // CUDA-core kernel otherwise)
  const bool tensor_jac = use_tensor_jacobian(p, n_src, n_rec);
  // tensor path: the quadrature weight w_k rides on the source fields (phi'_{s,k} = w_k phi_{s,k}),
  // which takes one complex product per A element out of the kernel's arrow transform
  if (tensor_jac)
    for (int s = 0; s < n_src; ++s)
      for (int k = 0; k < ns; ++k) scale[(size_t)s * ns + k] = cmul(scale[(size_t)s * ns + k], d2(weights[k]));
  DeviceBuffer dscale(sizeof(double2) * scale.size(), st);
  LT_CUDA(cudaMemcpyAsync(dscale.get(), scale.data(), sizeof(double2) * scale.size(), cudaMemcpyHostToDevice, st));
  DeviceBuffer fields(sizeof(double2) * (size_t)B * ns * n, st);
  {
    TraceScope tr(ctx, "  expand", B);
    expand_solutions(p, res, dscale.as<double2>(), fields.as<double2>(), tensor_jac);
  }
  res.U.clear();  // free the bases before the slice

  std::vector<double2> w(ns), wz(ns);
  for (int k = 0; k < ns; ++k) {
    // tensor path: w_k is already in the source fields (w = 1 for the predictions, wz = z_k or 1)
    w[k] = tensor_jac ? make_double2(1.0, 0.0) : d2(weights[k]);
    const cd zf = ex.storativity_z_factor ? nodes[k] : cd(1.0, 0.0);
    wz[k] = d2(tensor_jac ? zf : weights[k] * zf);
  }
  DeviceBuffer dw(sizeof(double2) * 2 * ns, st);
  LT_CUDA(cudaMemcpyAsync(dw.get(), w.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dw.as<double2>() + ns, wz.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));

  if (jac_out && p->kind == LT_GRID_P1_TRI) {
    TraceScope tr(ctx, "  jacobian_p1", B);
    const int nx = p->levels[0]->nx, nc = nx + 1;
    const int64_t nelem = 2 * (int64_t)nc * nc;
    const int64_t n_param = ex.include_storativity ? 2 * nelem : nelem;
    double* J = jac_out;
    DeviceBuffer jtmp;
    if (mem != LT_MEM_DEVICE) {
      jtmp.allocate(sizeof(double) * (size_t)n_src * n_rec * n_param, st);
      J = jtmp.as<double>();
    }
    const int nsub_r = (n_rec + RB - 1) / RB;
    const int nsub_total = ((n_src + SB - 1) / SB) * nsub_r;
    LT_REQUIRE(nsub_total <= kT / 2, "jacobian: too many source/receiver blocks for one CTA (n_src*n_rec too large)");
    int TC = std::max(1, kT / (2 * nsub_total));
    TC = std::min(TC, nc);
    auto smem_for = [&](int tc) { return sizeof(double2) * (size_t)4 * B * 2 * tc + sizeof(double) * 4 * tc; };
    while (TC > 1 && smem_for(TC) > 110 * 1024) TC /= 2;
    const size_t smem = smem_for(TC);
    const int tiles_x = (nc + TC - 1) / TC;
    LT_CUDA(cudaFuncSetAttribute(jacobian_p1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double h = p->grid.h;
    const double bytes = (double)n * 16.0 * ns * B + (double)nelem * 8.0 * n_src * n_rec * (ex.include_storativity ? 2 : 1);
    launch(ctx, "jacobian", bytes, [&] {
      jacobian_p1_kernel<<<(unsigned)(tiles_x * (int64_t)nc), kT, smem, st>>>(
          nx, h * h, p->kappa.as<double>(), p->storativity.as<double>(), fields.as<double2>(), n_src, n_rec, ns,
          dw.as<double2>(), dw.as<double2>() + ns, TC, tiles_x, nsub_r, nsub_total, J,
          ex.include_storativity ? J + nelem : nullptr, n_param);
    });
    if (mem != LT_MEM_DEVICE)
      LT_CUDA(cudaMemcpyAsync(jac_out, J, sizeof(double) * (size_t)n_src * n_rec * n_param, cudaMemcpyDeviceToHost, st));
  } else if (jac_out) {
    TraceScope tr(ctx, "  jacobian", B);
    const int64_t n_param = ex.include_storativity ? 2 * n : n;
    double* J = jac_out;
    DeviceBuffer jtmp;
    if (mem != LT_MEM_DEVICE) {
      jtmp.allocate(sizeof(double) * (size_t)n_src * n_rec * n_param, st);
      J = jtmp.as<double>();
    }
    fd_jacobian_kernels(p, p->view(0), p->kappa.as<double>(), p->storativity.as<double>(), fields.as<double2>(), n_src,
                        n_rec, ns, dw.as<double2>(), tensor_jac, ex.include_storativity != 0, J, n_param, n);
    if (mem != LT_MEM_DEVICE)
      LT_CUDA(cudaMemcpyAsync(jac_out, J, sizeof(double) * (size_t)n_src * n_rec * n_param, cudaMemcpyDeviceToHost, st));
  }
  if (pred_out) {
    DeviceBuffer didx(sizeof(int64_t) * rec.idx.size(), st), dwt(sizeof(double) * rec.w.size(), st),
        dcnt(sizeof(int) * rec.cnt.size(), st), dout(sizeof(double) * (size_t)n_src * n_rec, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), rec.idx.data(), sizeof(int64_t) * rec.idx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dwt.get(), rec.w.data(), sizeof(double) * rec.w.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), rec.cnt.data(), sizeof(int) * rec.cnt.size(), cudaMemcpyHostToDevice, st));
    launch(ctx, "predict", 0.0, [&] {
      predict_kernel<<<blocks_for((int64_t)n_src * n_rec, 128), 128, 0, st>>>(n, n_src, n_rec, ns, fields.as<double2>(),
                                                                             dw.as<double2>(), didx.as<int64_t>(),
                                                                             dwt.as<double>(), dcnt.as<int>(), dout.as<double>(), tensor_jac ? 1 : 0);
    });
    LT_CUDA(cudaMemcpyAsync(pred_out, dout.get(), sizeof(double) * (size_t)n_src * n_rec, cudaMemcpyDeviceToHost, st));
  }
  stream_sync(ctx);
}


// ---- the split build of one Jacobian time slice -----------------------
// Items (sources, then receivers) are partitioned over ranks; each rank solves its items'
// shifted families (split_solve), exports the rows of its bases that every z-slab (with a
// one-plane halo) needs (split_export: the caller's all-to-all moves them, NCCL over NVLink),
// and assembles the J columns of its own slab from every item's slab bases
// (jacobian_assemble_slab).  J rows never need a reduction; each (s, r) pair's row is split by
// columns only.
namespace {

// pred[s r_count + r] = 2 Re sum_k c_{s,k} sum_q wt_q sum_j Y[s,k,j] U_j[s][idx_q]
__global__ void basis_predict_kernel(int64_t n, int n_src, int n_rec, int ns, const double2* const* __restrict__ cols,
                                     const double2* __restrict__ Y, int ystride, const int* __restrict__ m_used,
                                     const double2* __restrict__ c, const int64_t* __restrict__ idx,
                                     const double* __restrict__ wt, const int* __restrict__ cnt, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_src * n_rec) return;
  const int s = t / n_rec, r = t % n_rec;
  double2 acc = make_double2(0.0, 0.0);
  for (int k = 0; k < ns; ++k) {
    const int bk = s * ns + k;
    double2 v = make_double2(0.0, 0.0);
    for (int j = 0; j < m_used[bk]; ++j) {
      double2 u = make_double2(0.0, 0.0);
      for (int q = 0; q < cnt[r]; ++q) u = cadd(u, cscale(cols[j][(int64_t)s * n + idx[r * 8 + q]], wt[r * 8 + q]));
      v = cfma(Y[(int64_t)bk * ystride + j], u, v);
    }
    acc = cfma(c[bk], v, acc);
  }
  out[t] = 2.0 * acc.x;
}

}  // namespace

void split_solve(lt_split_s* sp) {
  lt_pencil p = sp->p;
  LT_REQUIRE(p->kind == LT_GRID_FD_CELL && !p->from_csr, "split build: FD grid pencils with parameter fields only");
  const lt_experiment& ex = sp->ex;
  LT_REQUIRE(ex.n_src >= 1 && ex.n_rec >= 1 && sp->t >= 0 && sp->t < ex.n_times, "split build: bad experiment / time");
  LT_REQUIRE(ex.n_quad >= 4 && ex.n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
  talbot_build(ex.n_quad, ex.times[sp->t], ex.contour, nullptr, &sp->nodes, nullptr, &sp->weights);
  solve_slice_items(p, ex, sp->nodes, sp->item0, sp->item1, sp->res);
}

void split_export(lt_split_s* sp, int plane0, int plane1, int m_pad, double2* dst, int mem) {
  lt_pencil p = sp->p;
  cudaStream_t st = p->ctx->stream;
  const LevelView L = p->view(0);
  const int nplanes = p->dim == 3 ? L.nz : L.ny;
  const int64_t plane = p->dim == 3 ? (int64_t)L.nx * L.ny : L.nx;
  LT_REQUIRE(0 <= plane0 && plane0 < plane1 && plane1 <= nplanes, "split export: bad plane range");
  const int B = sp->item1 - sp->item0, ncols = (int)sp->res.U.size();
  LT_REQUIRE(m_pad >= ncols, "split export: m_pad below this part's basis columns");
  const int64_t cells = (int64_t)(plane1 - plane0) * plane;
  const auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (int j = 0; j < m_pad; ++j) {
    double2* d = dst + (int64_t)j * B * cells;
    if (j < ncols) {
      LT_CUDA(cudaMemcpy2DAsync(d, sizeof(double2) * cells, sp->res.U[j].as<double2>() + plane0 * plane,
                                sizeof(double2) * p->n, sizeof(double2) * cells, B, kind, st));
    } else if (mem == LT_MEM_DEVICE) {
      LT_CUDA(cudaMemsetAsync(d, 0, sizeof(double2) * B * cells, st));
    } else {
      std::memset(d, 0, sizeof(double2) * B * cells);
    }
  }
  stream_sync(p->ctx);
}

void split_coefficients(lt_split_s* sp, double2* Y, int* m_used, int m_pad) {
  cudaStream_t st = sp->p->ctx->stream;
  const OuterResult& res = sp->res;
  const int B = res.B, ns = res.n_shifts;
  std::vector<double2> Yd((size_t)B * ns * res.maxit);
  LT_CUDA(cudaMemcpyAsync(Yd.data(), res.Y.get(), sizeof(double2) * Yd.size(), cudaMemcpyDeviceToHost, st));
  stream_sync(sp->p->ctx);
  for (int bk = 0; bk < B * ns; ++bk) {
    const int mu = res.m_used[bk];
    LT_REQUIRE(mu <= m_pad, "split coefficients: m_pad below this part's basis columns");
    m_used[bk] = mu;
    for (int j = 0; j < m_pad; ++j) Y[(size_t)bk * m_pad + j] = j < mu ? Yd[(size_t)bk * res.maxit + j] : make_double2(0, 0);
  }
}

void split_predictions(lt_split_s* sp, double* out) {
  lt_pencil p = sp->p;
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const lt_experiment& ex = sp->ex;
  const int s_end = std::min(sp->item1, ex.n_src);
  const int n_loc = std::max(0, s_end - sp->item0);  // this part's sources: local items [0, n_loc)
  if (n_loc == 0) return;
  const OuterResult& res = sp->res;
  const int ns = res.n_shifts;
  std::vector<double2> c((size_t)n_loc * ns);
  for (int s = 0; s < n_loc; ++s)
    for (int k = 0; k < ns; ++k)
      c[(size_t)s * ns + k] = d2(sp->weights[k] * (ex.rates[sp->item0 + s] / sp->nodes[k]));
  const PointSet rec = make_points(p, ex.receivers, ex.n_rec);
  std::vector<const double2*> cols(std::max<size_t>(res.U.size(), 1), nullptr);
  for (size_t j = 0; j < res.U.size(); ++j) cols[j] = res.U[j].as<double2>();
  DeviceBuffer dcols(sizeof(void*) * cols.size(), st), dmu(sizeof(int) * res.m_used.size(), st),
      dc(sizeof(double2) * c.size(), st), didx(sizeof(int64_t) * rec.idx.size(), st),
      dwt(sizeof(double) * rec.w.size(), st), dcnt(sizeof(int) * rec.cnt.size(), st),
      dout(sizeof(double) * (size_t)n_loc * ex.n_rec, st);
  LT_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(void*) * cols.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dmu.get(), res.m_used.data(), sizeof(int) * res.m_used.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dc.get(), c.data(), sizeof(double2) * c.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(didx.get(), rec.idx.data(), sizeof(int64_t) * rec.idx.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dwt.get(), rec.w.data(), sizeof(double) * rec.w.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dcnt.get(), rec.cnt.data(), sizeof(int) * rec.cnt.size(), cudaMemcpyHostToDevice, st));
  launch(ctx, "predict", 0.0, [&] {
    basis_predict_kernel<<<blocks_for((int64_t)n_loc * ex.n_rec, 128), 128, 0, st>>>(
        p->n, n_loc, ex.n_rec, ns, dcols.as<const double2*>(), res.Y.as<double2>(), res.maxit, dmu.as<int>(),
        dc.as<double2>(), didx.as<int64_t>(), dwt.as<double>(), dcnt.as<int>(), dout.as<double>());
  });
  LT_CUDA(cudaMemcpyAsync(out, dout.get(), sizeof(double) * (size_t)n_loc * ex.n_rec, cudaMemcpyDeviceToHost, st));
  stream_sync(ctx);
}

void jacobian_assemble_slab(lt_pencil p, const lt_experiment& ex, int t, int plane0, int plane1, int halo_lo,
                            int halo_hi, const double2* U, int m, const double2* Y, const int* m_used, int mem,
                            double* jac_out) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  LT_REQUIRE(p->kind == LT_GRID_FD_CELL && !p->from_csr, "split build: FD grid pencils with parameter fields only");
  LT_REQUIRE(t >= 0 && t < ex.n_times && ex.n_quad >= 4 && ex.n_quad % 2 == 0, "split build: bad time / n_quad");
  LevelView L = p->view(0);
  const int nplanes = p->dim == 3 ? L.nz : L.ny;
  const int64_t plane = p->dim == 3 ? (int64_t)L.nx * L.ny : L.nx;
  LT_REQUIRE(0 <= plane0 && plane0 < plane1 && plane1 <= nplanes, "assemble slab: bad plane range");
  LT_REQUIRE(halo_lo == (plane0 > 0 ? 1 : 0) && halo_hi == (plane1 < nplanes ? 1 : 0),
             "assemble slab: one halo plane on each interior side");
  LT_REQUIRE(m >= 1, "assemble slab: no basis columns");
  const int n_src = ex.n_src, n_rec = ex.n_rec, B = n_src + n_rec, ns = ex.n_quad / 2;
  const int ps = plane0 - halo_lo, V = plane1 + halo_hi - ps;
  const int64_t n_view = (int64_t)V * plane, n_slab = (int64_t)(plane1 - plane0) * plane;
  std::vector<cd> nodes, weights;
  talbot_build(ex.n_quad, ex.times[t], ex.contour, nullptr, &nodes, nullptr, &weights);
  // the slab's view of the fine level: planes [ps, ps + V)
  LevelView Lv = L;
  if (p->dim == 3) {
    Lv.nz = V;
    Lv.Tx += (int64_t)ps * L.ny * (L.nx + 1);
    Lv.Ty += (int64_t)ps * (L.ny + 1) * L.nx;
    Lv.Tz += (int64_t)ps * plane;
  } else {
    Lv.ny = V;
    Lv.Tx += (int64_t)ps * (L.nx + 1);
    Lv.Ty += (int64_t)ps * L.nx;
  }
  Lv.M += (int64_t)ps * plane;
  Lv.n = n_view;
  Lv.tiles_y = (Lv.ny + Lv.th - 1) / Lv.th;
  Lv.ntiles = Lv.tiles_x * Lv.tiles_y * Lv.nz;
  // the slab bases of all B items and their coefficients
  DeviceBuffer ubuf;
  const double2* Ud = U;
  if (mem != LT_MEM_DEVICE) {
    ubuf.allocate(sizeof(double2) * (size_t)m * B * n_view, st);
    LT_CUDA(cudaMemcpyAsync(ubuf.get(), U, ubuf.bytes(), cudaMemcpyHostToDevice, st));
    Ud = ubuf.as<double2>();
  }
  std::vector<const double2*> cols(m);
  for (int j = 0; j < m; ++j) cols[j] = Ud + (int64_t)j * B * n_view;
  DeviceBuffer dY(sizeof(double2) * (size_t)B * ns * m, st);
  LT_CUDA(cudaMemcpyAsync(dY.get(), Y, dY.bytes(), cudaMemcpyHostToDevice, st));
  std::vector<int> mu(m_used, m_used + (size_t)B * ns);
  const bool tensor_jac = use_tensor_jacobian(p, n_src, n_rec);
  std::vector<double2> scale((size_t)B * ns, make_double2(1.0, 0.0));
  for (int s = 0; s < n_src; ++s)
    for (int k = 0; k < ns; ++k) {
      const cd f = ex.rates[s] / nodes[k];
      scale[(size_t)s * ns + k] = d2(tensor_jac ? f * weights[k] : f);
    }
  DeviceBuffer dscale(sizeof(double2) * scale.size(), st);
  LT_CUDA(cudaMemcpyAsync(dscale.get(), scale.data(), sizeof(double2) * scale.size(), cudaMemcpyHostToDevice, st));
  DeviceBuffer fields(sizeof(double2) * (size_t)B * ns * n_view, st);
  expand_raw(ctx, n_view, B, ns, cols, dY.as<double2>(), m, mu, dscale.as<double2>(), fields.as<double2>(), tensor_jac);
  std::vector<double2> w(ns), wz(ns);
  for (int k = 0; k < ns; ++k) {
    w[k] = tensor_jac ? make_double2(1.0, 0.0) : d2(weights[k]);
    const cd zf = ex.storativity_z_factor ? nodes[k] : cd(1.0, 0.0);
    wz[k] = d2(tensor_jac ? zf : weights[k] * zf);
  }
  DeviceBuffer dw(sizeof(double2) * 2 * ns, st);
  LT_CUDA(cudaMemcpyAsync(dw.get(), w.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dw.as<double2>() + ns, wz.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));
  // J over the view (halo planes included), then the slab's columns of both blocks
  const int pairs = n_src * n_rec;
  const bool inc_s = ex.include_storativity != 0;
  const int64_t ldv = inc_s ? 2 * n_view : n_view;
  DeviceBuffer jv(sizeof(double) * (size_t)pairs * ldv, st);
  fd_jacobian_kernels(p, Lv, p->kappa.as<double>() + (int64_t)ps * plane, p->storativity.as<double>() + (int64_t)ps * plane,
                      fields.as<double2>(), n_src, n_rec, ns, dw.as<double2>(), tensor_jac, inc_s, jv.as<double>(), ldv,
                      n_view);
  const int64_t lds = inc_s ? 2 * n_slab : n_slab;
  const auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (int blk = 0; blk < (inc_s ? 2 : 1); ++blk)
    LT_CUDA(cudaMemcpy2DAsync(jac_out + blk * n_slab, sizeof(double) * lds,
                              jv.as<double>() + blk * n_view + (int64_t)halo_lo * plane, sizeof(double) * ldv,
                              sizeof(double) * n_slab, pairs, kind, st));
  stream_sync(ctx);
}

}  // namespace lt
