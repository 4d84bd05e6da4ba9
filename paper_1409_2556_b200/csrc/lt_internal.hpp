// Internal C++ types of the laptomo B200 library (not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "lt_common.cuh"

namespace lt {

// ---- device block cache -----------------------------------------------------------------
// Every buffer of a context lives on the context's single stream, so a freed block can be
// handed to the next request of the same rounded size on that stream with no driver call and
// no synchronisation (stream order is the only order).  The solver's request sizes repeat
// exactly from one time slice / build to the next (one vector per item, basis columns, the
// multigrid hierarchy, the field slab), so after the first slice it never touches the driver:
// growing the stream-ordered pool instead costs 15 ms - 1.7 s of host time per large request.
// On an out-of-memory the cache is returned to the pool and the request retried.  (allocator.cu)
void* cache_alloc(size_t bytes, cudaStream_t s);
void cache_free(void* p, size_t bytes, cudaStream_t s);
void cache_release_stream(cudaStream_t s);  // return a stream's cached blocks to the pool
size_t cache_cached_bytes();
uint64_t cache_driver_epoch();                // bytes held in free lists

// ---- stream-ordered device buffer -------------------------------------------------------
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(size_t bytes, cudaStream_t s) { allocate(bytes, s); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept { swap(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) { release(); swap(o); }
    return *this;
  }
  void allocate(size_t bytes, cudaStream_t s) {
    release();
    stream_ = s;
    bytes_ = bytes;
    if (bytes == 0) return;
    ptr_ = cache_alloc(bytes, s);
  }
  void ensure(size_t bytes, cudaStream_t s) {
    if (bytes > bytes_) allocate(bytes, s);
  }
  void release() {
    if (ptr_) cache_free(ptr_, bytes_, stream_);
    ptr_ = nullptr;
    bytes_ = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(ptr_); }
  size_t bytes() const { return bytes_; }
  void* get() const { return ptr_; }

 private:
  void swap(DeviceBuffer& o) {
    std::swap(ptr_, o.ptr_);
    std::swap(bytes_, o.bytes_);
    std::swap(stream_, o.stream_);
  }
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t stream_ = nullptr;
};

struct ProfileEntry {
  double ms = 0.0;
  int64_t launches = 0;
  double bytes = 0.0;
};

struct PendingEvent {
  std::string name;
  cudaEvent_t start, stop;
  double bytes;
  int tag;  // >= 0: bytes still to be scaled by the active-item fraction of step `tag` (inner.cu)
};

}  // namespace lt

// Host-visible convergence state of the device-resident COCG loop (inner.cu): a ring of
// kFlagRing slots in mapped pinned memory written by the control kernel, each slot paired with
// an event; the host reads slot it - kFlagLag while iteration it is still queued.
constexpr int kFlagRing = 4, kFlagLag = 1;
// The inner shift-and-invert solve is accepted at a relative residual of kInnerFloor x its
// tolerance (1e-11 by default): converged at the tolerance, or stagnated at the rounding floor
// within this margin.  Anything above would break the outer method's Arnoldi relation
// (K + tau_j M) u_j = v_j at the 1e-10 level of the shifts' own tolerance.
constexpr double kInnerFloor = 10.0;
struct FlagSlot {
  double worst;  // max over the items still iterating of ||r||^2 / (tol^2 ||v||^2)
  int active;    // items still iterating
  int pad;
};

struct lt_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  int64_t launches = 0;
  std::map<std::string, lt::ProfileEntry> profile;
  std::vector<lt::PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  int num_sms = 148;
  int sample_every = 1;                              // time 1 in N launches of each class
  std::map<const char*, int64_t> class_counter;      // keyed by the (literal) class name
  // >= 0 inside a device-resident loop: launches record this tag, and their algorithmic bytes
  // (written for every item of the batch) are scaled once the loop knows how many items were
  // still active at that step
  int profile_tag = -1;
  // host gap accounting: wall time from the return of a stream synchronisation (the stream is
  // empty) to the next kernel launch -- the GPU is idle for at least that long
  bool drained = false;
  std::chrono::steady_clock::time_point drain_t{};
  double gap_ms = 0.0;
  // cached driver-side free memory (available_device_bytes)
  bool mem_probe_valid = false;
  double mem_probe = 0.0;
  uint64_t mem_probe_epoch = 0;
  std::chrono::steady_clock::time_point mem_probe_t{};
  int64_t gap_count = 0;

  cusolverDnHandle_t solver = nullptr;  // dense LU of the coarsest multigrid levels (lazy)
  cusolverDnHandle_t solver_handle();
  FlagSlot* flag_host = nullptr;  // mapped pinned ring (kFlagRing slots)
  FlagSlot* flag_dev = nullptr;   // its device alias
  cudaEvent_t flag_ev[kFlagRing] = {};
  FlagSlot* flag_ring_dev();      // allocates the ring and its events on first use
  volatile FlagSlot* flag_ring_host() { return flag_host; }

  void resolve_profile();    // waits for all pending events
  void resolve_completed();  // accumulates the already-completed prefix of pending events
  cudaEvent_t take_event();
};

namespace lt {

// LT_DEBUG_SYNC=1: synchronise after every launch and name the kernel class that failed
inline bool debug_sync() {
  static const bool on = std::getenv("LT_DEBUG_SYNC") != nullptr;
  return on;
}
// Launch a kernel (callable issuing exactly one launch on ctx->stream) with accounting.
inline void stream_sync(lt_ctx ctx) {
  LT_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->drain_t = std::chrono::steady_clock::now();
  ctx->drained = true;
}
template <class F>
inline void launch(lt_ctx ctx, const char* name, double algorithmic_bytes, F&& f) {
  ctx->launches++;
  if (ctx->drained) {
    const double gap = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ctx->drain_t).count();
    ctx->gap_ms += gap;
    ctx->gap_count++;
    ctx->drained = false;
    static const bool gap_trace = std::getenv("LT_GAPTRACE") != nullptr;  // diagnostics: name the long gaps
    if (gap_trace && gap > 0.3) std::fprintf(stderr, "[lt] host gap %8.3f ms before %s\n", gap, name);
  }
  if (ctx->profiling && (ctx->class_counter[name]++ % ctx->sample_every) == 0) {
    cudaEvent_t a = ctx->take_event(), b = ctx->take_event();
    cudaEventRecord(a, ctx->stream);
    f();
    cudaEventRecord(b, ctx->stream);
    ctx->pending.push_back({name, a, b, algorithmic_bytes, ctx->profile_tag});
    check_launch(name);
    if (ctx->pending.size() >= 1024 && ctx->profile_tag < 0) ctx->resolve_completed();  // non-blocking
    return;
  }
  f();
  check_launch(name);
  if (debug_sync()) {
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) throw Error(LT_ERR_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
  }
}

// ---- host-side phase tracing (LT_TRACE=1): synchronising wall-clock scopes on stderr ----
inline bool trace_on() {
  static const bool on = std::getenv("LT_TRACE") != nullptr;
  return on;
}

class TraceScope {
 public:
  TraceScope(lt_ctx ctx, const char* what, int arg = -1) : ctx_(ctx), what_(what), arg_(arg) {
    if (trace_on()) {
      cudaStreamSynchronize(ctx_->stream);
      t0_ = std::chrono::steady_clock::now();
    }
  }
  ~TraceScope() {
    if (!trace_on()) return;
    cudaStreamSynchronize(ctx_->stream);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    std::fprintf(stderr, "[lt] %-22s %4d %10.3f ms\n", what_, arg_, ms);
  }

 private:
  lt_ctx ctx_;
  const char* what_;
  int arg_;
  std::chrono::steady_clock::time_point t0_{};
};

// ---- discretisation levels -----------------------------------------------------------
// Cell-centred FD level: face transmissibilities including the Dirichlet boundary faces,
//   Tx[(k*ny + j)*(nx+1) + i]  face between cells i-1 and i (i = 0, nx: boundary)
//   Ty[(k*(ny+1) + j)*nx + i]  face between rows j-1 and j
//   Tz[(k*ny + j)*nx + i]      face between planes k-1 and k  (k in [0, nz])
//   M[a]                       diagonal mass (S h^d, summed on coarse levels)
// Storage type of Level::packrb.  bfloat16 (default): the colour-split V-cycle is then the exact
// V-cycle of the operator A' whose faces and masses are the bf16 roundings of A's -- every
// face term of K and every mass is perturbed by a relative 2^-9 at most, so A' is spectrally
// equivalent to A within (1 +- 0.002) and as good a COCG preconditioner as the FP32 one
// (same iteration counts), symmetric as before -- while the coefficient tiles, half of what
// a half sweep's CTA pulls from L2, shrink to half: a 7-deep plane ring fits where 5 did.
#ifndef RB_BF16
#define RB_BF16 1
#endif
#if RB_BF16
typedef unsigned short rb_coef_t;
#else
typedef float rb_coef_t;
#endif

struct Level {
  int nx = 1, ny = 1, nz = 1;
  int64_t n = 0;
  double* Tx = nullptr;
  double* Ty = nullptr;
  double* Tz = nullptr;
  double* M = nullptr;
  // P1 only: positive mass couplings of the 7-point M (E/W edges like Tx, N/S like Ty, the
  // NE neighbour stored at the node); null for FD (diagonal M)
  double* Mx = nullptr;
  double* My = nullptr;
  double* Md = nullptr;
  DeviceBuffer storage;
  // FP32 copy of the same arrays (same layout) for the mixed-precision V-cycle
  float* Tx32 = nullptr;
  float* Ty32 = nullptr;
  float* Tz32 = nullptr;
  float* M32 = nullptr;
  float* Mx32 = nullptr;
  float* My32 = nullptr;
  float* Md32 = nullptr;
  DeviceBuffer storage32;
  DeviceBuffer elem;       // P1: per-element kappa then S on this level (coarsening input)
  // FD: per-cell packed {west face, south face, bottom face, mass} over (nx+1) x (ny+1) x
  // (nz+1) (the high boundary faces in the extra row / column / plane): pack32 (FP32
  // records) for the natural-layout TMA kernels, pack64 (FP64, finest level, planar
  // [k][j][comp][i] with rows of nx + 2) for the COCG operator
  DeviceBuffer pack32, pack64;
  // FD levels with nx % 4 == 0 and nx >= 64: the coefficients in the colour-split layout of
  // the red-black TMA kernels (inner.cu), [k][j][comp W,S,B,M][colour][pos] with pos = i / 2,
  // colour = (i + j + k) & 1, rb_P >= nx / 2 + 1 positions per colour (padded to a multiple
  // of 8), stored as rb_coef_t
  DeviceBuffer packrb;
  int rb_P = 0;
  int agg[3] = {1, 1, 1};  // aggregation to the next coarser level (FD)
};

// Device view of a level passed by value to kernels (R = double: the operator; R = float:
// the preconditioner copy).
template <class R>
struct LevelViewT {
  int nx, ny, nz, dim;
  int64_t n;
  const R* Tx;
  const R* Ty;
  const R* Tz;
  const R* M;
  // 256-thread (x, y) tiles: tw x th cells, tw a power of two (tws = log2 tw)
  int tw, tws, th, tiles_x, tiles_y, ntiles;
  const R* Mx;  // P1 mass couplings (null for FD)
  const R* My;
  const R* Md;
  // vectors of this level are stored colour-split (inner.cu: rb_index); set by the V-cycle
  int split;
};
using LevelView = LevelViewT<double>;
using LevelView32 = LevelViewT<float>;

struct CoarseFactor {
  double2 tau;
  DeviceBuffer inverse;    // [A | A^{-1}] n_c x 2n_c complex128, row-major (Gauss-Jordan work)
  DeviceBuffer inverse32;  // A^{-1} n_c x n_c complex64, row-major (V-cycle coarsest solve)
};

// Exact banded LU of K + tau M for 2-D pencils (band.cu), LAPACK zgbtrf layout
struct BandFactor {
  double2 tau;
  int64_t n = 0;
  int kl = 0, ku = 0, ldab = 0;
  DeviceBuffer ab;    // ldab x n complex128
  DeviceBuffer ipiv;  // n pivots + info
};

// Per-solve FGMRES basis kept for keep_basis queries.
struct KeptBasis {
  int n_rhs = 0;
  std::vector<int> steps;
  std::vector<double> beta;
  std::vector<std::vector<double2>> V, U, H, taus;  // per rhs
};

}  // namespace lt

struct lt_pencil_s {
  lt_ctx ctx = nullptr;
  lt_grid grid{};
  int dim = 2;
  int kind = LT_GRID_FD_CELL;
  int64_t n = 0;
  std::vector<std::unique_ptr<lt::Level>> levels;
  std::vector<std::unique_ptr<lt::CoarseFactor>> factors;  // keyed by exact tau
  std::vector<std::unique_ptr<lt::BandFactor>> band_factors;  // exact banded LU, keyed by exact tau
  std::vector<double2> band_taus;  // shifts whose inner solve needs the banded direct solve
  lt::DeviceBuffer kappa;         // per cell (fine), for Jacobian
  lt::DeviceBuffer storativity;   // per cell (fine)
  bool from_csr = false;          // built by lt_pencil_create_csr: no parameter fields
  double inner_tol = 1e-12;
  int inner_maxit = 200;
  lt::KeptBasis kept;
  cudaGraphExec_t inner_exec = nullptr;  // the inner COCG iteration body (updated per chunk)
  cudaGraphExec_t graph_exec(cudaGraph_t g);  // instantiates or updates inner_exec to g
  lt_pencil_s() = default;
  lt_pencil_s(const lt_pencil_s&) = delete;
  lt_pencil_s& operator=(const lt_pencil_s&) = delete;
  ~lt_pencil_s();

  lt::LevelView view(int l) const;
  lt::LevelView32 view32(int l) const;
  const lt::CoarseFactor& factor(double2 tau);  // prepares on miss
};

namespace lt {

// pencil.cu
void pencil_build(lt_pencil p, const double* log_kappa, const double* log_s, int mem);
void pencil_build_csr(lt_pencil p, const lt_sparse* K, const lt_sparse* M);
void apply_batch(lt_pencil p, int level, const double2* taus_dev, const double2* x, int64_t xs,
                 double2* y, int64_t ys, int B, bool mass_only, const char* name);
void point_weights(const lt_pencil_s* p, const double* point, int64_t* idx, double* w, int* count);

// inner.cu: u_b = (K + tau_b M)^{-1} v_b, b < B, strided vectors; taus on host.
// Tiled TMA tensor map over 8-byte elements (no swizzle, out-of-bounds boxes read as zero);
// dims / box innermost first, strides_bytes for dims 1.. (tma.cu)
CUtensorMap tma_map_8b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box);
// the same over 4-byte (FP32) elements.  Every box must start 16-byte aligned in its
// innermost dimension: an unaligned start faults ("illegal instruction") on B200.
CUtensorMap tma_map_4b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box);
CUtensorMap tma_map_2b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box);

// device bytes a solve may still take: free + the pool's reserved-but-unused memory (ctx.cu)
double available_device_bytes(lt_ctx ctx);

// active (device, B ints) may be null: items with active[b] == 0 are skipped (u untouched);
// rel_out (host, B) may be null: each item's final relative residual ||v - A u|| / ||v||
// (recursive COCG residual).
void inner_solve(lt_pencil p, int B, const double2* taus_host, const double2* v, int64_t vs,
                 double2* u, int64_t us, const int* active = nullptr, double* rel_out = nullptr);

// band.cu: the exact banded shift-and-invert of 2-D pencils
bool band_feasible(const lt_pencil_s* p);
const BandFactor& pencil_band_factor(lt_pencil p, double2 tau);
void band_solve(lt_pencil p, const BandFactor& f, int B, const double2* v, int64_t vs, double2* u, int64_t us);

// fgmres.cu
struct OuterProblem {
  int B = 0;           // items (right-hand sides) in lockstep
  int n_shifts = 0;
  const double2* b = nullptr;  // device, B x n
  std::vector<double2> shifts;        // B * n_shifts (host)
  std::vector<std::vector<double2>> tau_table;  // per item: tau applied at iteration j
  int variant = LT_VARIANT_GMRES;
  double tol = 1e-10;
  int maxit = 0;
  bool record_history = false;
  bool keep_basis = false;
};

struct OuterResult {
  int B = 0, n_shifts = 0, cap = 0;
  std::vector<int> iterations;             // per item
  std::vector<lt_shift_status> status;     // B * n_shifts
  std::vector<double> history;             // B * n_shifts * maxit (if recorded)
  int maxit = 0;
  // Basis form of the solutions: x_{b,k} = U_b[:, :m_bk] y_{b,k}
  std::vector<DeviceBuffer> U;             // per column j: B x n
  DeviceBuffer Y;                          // B * n_shifts * cap complex (device)
  std::vector<int> m_used;                 // B * n_shifts: number of columns in y
};

void outer_solve(lt_pencil p, const OuterProblem& prob, OuterResult& res);

// x_out[b][k] = scale[b][k] * U_b y_{b,k}  (device output, B * n_shifts * n)
// cell_major: out[(k n + a) B + b] instead of out[(b ns + k) n + a]
void expand_solutions(lt_pencil p, const OuterResult& res, const double2* scale_dev,
                      double2* x_out, bool cell_major = false);
// the same from raw bases: cols[j] = column j (B items of n cells each, item stride n),
// Y[(b ns + k) ystride + j] (device), m_used (host, B ns)
void expand_raw(lt_ctx ctx, int64_t n, int B, int ns, const std::vector<const double2*>& cols, const double2* Y,
                int ystride, const std::vector<int>& m_used, const double2* scale_dev, double2* x_out,
                bool cell_major);

}  // namespace lt

// one rank's part of a split Jacobian time slice (drivers.cu)
struct lt_split_s {
  lt_pencil p = nullptr;
  int t = 0, item0 = 0, item1 = 0;
  std::vector<double> sources, receivers, rates, times;  // copies of the experiment's arrays
  lt_experiment ex{};                                     // pointing into them
  std::vector<std::complex<double>> nodes, weights;
  lt::OuterResult res;
};
