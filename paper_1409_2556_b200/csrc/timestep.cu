// SURVEY.md §8f row 4 on the device: the Crank-Nicolson reference integrator
// (crank_nicolson, forward.cpp:200-258) and the 1-norm condition estimate of a shifted pencil
// (estimate_norm_1 / estimate_condition_1norm, condest.cpp:11-49).
//
// Crank-Nicolson: (M + dt/2 K) h_{n+1} = (M - dt/2 K) h_n + dt q b.  Multiplying by 2/dt,
//   (K + tau M) h_{n+1} = -(K - tau M) h_n + 2 q b,   tau = 2 / dt  (real, positive),
// so one step is one pencil apply at z = -tau and one shift-and-invert solve at tau: the same
// matrix-free operator and multigrid-preconditioned inner solve as the Laplace path (the
// reference factors M + dt/2 K once with SimplicialLDLT; here the preconditioner hierarchy of
// tau is built once and every step's solve runs to the inner tolerance).  All n_src problems of a
// call step in lockstep.  Samples are recorded like the reference: at the step that reaches a
// sample time, linear interpolation between the two states around it (exact hits and t = 0 copy).
//
// Condition estimate: Hager's iteration (at most 6 steps) on A = K + z M with the forward and
// adjoint applies, and on A^{-1} with the shift-and-invert solve and its adjoint (the conjugate
// of the solve of the conjugate, K and M being real symmetric); the result is the product of
// the two 1-norm lower bounds, never above kappa_1(A).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "drivers.hpp"
#include "lt_internal.hpp"

namespace lt {

namespace {

constexpr int kT = 256;

// v = -(K - tau M) h + 2 q b   (y holds (K - tau M) h from apply_batch)
__global__ void cn_rhs_kernel(int64_t n, int B, const double2* __restrict__ y, const double* __restrict__ src,
                              const double* __restrict__ rates, double2* __restrict__ v) {
  const int b = blockIdx.y;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const double2 ya = y[b * n + a];
    v[b * n + a] = make_double2(-ya.x + 2.0 * rates[b] * src[b * n + a], -ya.y);
  }
}

// out[(b n_s + s) n + a] = (1 - w) Re hp + w Re h
__global__ void cn_record_kernel(int64_t n, int B, const double2* __restrict__ hp, const double2* __restrict__ h,
                                 double w, int s, int n_samples, double* __restrict__ out) {
  const int b = blockIdx.y;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    out[((int64_t)b * n_samples + s) * n + a] = (1.0 - w) * hp[b * n + a].x + w * h[b * n + a].x;
}

__global__ void real_to_complex_kernel(int64_t count, const double* __restrict__ in, double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_double2(in ? in[i] : 0.0, 0.0);
}

// per-block partial sums of |y| and the block's max |z| with its index
__global__ void __launch_bounds__(kT) l1_partial_kernel(int64_t n, const double2* __restrict__ y, double* __restrict__ part) {
  __shared__ double sh[kT / 32];
  double s = 0.0;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    s += hypot(y[a].x, y[a].y);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffff, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kT / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// xi = y / |y| (1 where y = 0)
__global__ void sign_kernel(int64_t n, const double2* __restrict__ y, double2* __restrict__ xi) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const double m = hypot(y[a].x, y[a].y);
    xi[a] = m == 0.0 ? make_double2(1.0, 0.0) : make_double2(y[a].x / m, y[a].y / m);
  }
}

// block max of |z| (first index on ties, like Eigen's maxCoeff)
__global__ void __launch_bounds__(kT) absmax_partial_kernel(int64_t n, const double2* __restrict__ z,
                                                            double* __restrict__ vmax, int64_t* __restrict__ imax) {
  __shared__ double sv[kT];
  __shared__ int64_t si[kT];
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const double m = hypot(z[a].x, z[a].y);
    if (m > best) { best = m; bi = a; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      const double ov = sv[threadIdx.x + s];
      const int64_t oi = si[threadIdx.x + s];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi >= 0 && (si[threadIdx.x] < 0 || oi < si[threadIdx.x]))) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    vmax[blockIdx.x] = sv[0];
    imax[blockIdx.x] = si[0];
  }
}

__global__ void conj_inplace_kernel(int64_t n, double2* __restrict__ x) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    x[a].y = -x[a].y;
}

unsigned grid_for(int64_t n, lt_ctx ctx) { return (unsigned)std::min<int64_t>(blocks_for(n, kT), 8 * ctx->num_sms); }

void check_inner_cn(lt_pencil p, const std::vector<double>& rel) {
  for (double r : rel)
    if (!(r <= kInnerFloor * p->inner_tol))
      throw Error(LT_ERR_PRECONDITIONER, "crank_nicolson: the shift-and-invert solve of M + dt/2 K did not converge "
                                         "(relative residual " + std::to_string(r) + ")");
}

}  // namespace

void crank_nicolson(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
                    double dt, const double* sample_times, int n_samples, int mem, double* out, int* steps_out) {
  LT_REQUIRE(dt > 0.0, "crank_nicolson: dt must be positive");
  LT_REQUIRE(n_samples >= 1 && sample_times, "crank_nicolson: no sample times");
  LT_REQUIRE(n_src >= 1 && sources && rates && out, "crank_nicolson: missing source");
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  const int B = n_src;
  const double t_end = *std::max_element(sample_times, sample_times + n_samples);
  const double tau = 2.0 / dt;
  const auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DeviceBuffer dsrc(sizeof(double) * (size_t)B * n, st), drates(sizeof(double) * B, st);
  LT_CUDA(cudaMemcpyAsync(dsrc.get(), sources, dsrc.bytes(), kind, st));
  LT_CUDA(cudaMemcpyAsync(drates.get(), rates, sizeof(double) * B, cudaMemcpyHostToDevice, st));
  DeviceBuffer state(sizeof(double2) * (size_t)B * n * 4, st);
  double2* h = state.as<double2>();
  double2* hp = h + (size_t)B * n;
  double2* y = hp + (size_t)B * n;
  double2* v = y + (size_t)B * n;
  DeviceBuffer ih;
  if (initial_head) {
    ih.allocate(sizeof(double) * (size_t)B * n, st);
    LT_CUDA(cudaMemcpyAsync(ih.get(), initial_head, ih.bytes(), kind, st));
  }
  const unsigned g1 = grid_for((int64_t)B * n, ctx);
  launch(ctx, "cn_vec", 16.0 * B * n, [&] {
    real_to_complex_kernel<<<g1, kT, 0, st>>>((int64_t)B * n, initial_head ? ih.as<double>() : nullptr, h);
  });
  DeviceBuffer dout;
  double* o = out;
  if (mem != LT_MEM_DEVICE) {
    dout.allocate(sizeof(double) * (size_t)B * n_samples * n, st);
    o = dout.as<double>();
  }
  std::vector<char> filled(n_samples, 0);
  const dim3 g2(std::max(1u, grid_for(n, ctx) / (unsigned)std::max(1, B)), B);
  auto record = [&](double t_prev, const double2* head_prev, double t_now, const double2* head_now) {
    for (int s = 0; s < n_samples; ++s) {
      if (filled[s]) continue;
      const double target = sample_times[s];
      if (target <= t_now + 1e-9 * dt) {
        double w = 1.0;
        if (!(std::fabs(target - t_now) <= 1e-9 * dt || t_now == t_prev)) w = (target - t_prev) / (t_now - t_prev);
        launch(ctx, "cn_vec", 24.0 * B * n, [&] {
          cn_record_kernel<<<g2, kT, 0, st>>>(n, B, head_prev, head_now, w, s, n_samples, o);
        });
        filled[s] = 1;
      }
    }
  };
  record(0.0, h, 0.0, h);
  DeviceBuffer dz(sizeof(double2) * B, st);
  std::vector<double2> zneg(B, make_double2(-tau, 0.0)), taus(B, make_double2(tau, 0.0));
  LT_CUDA(cudaMemcpyAsync(dz.get(), zneg.data(), sizeof(double2) * B, cudaMemcpyHostToDevice, st));
  int steps = 0;
  double t = 0.0;
  std::vector<double> rel(B);
  while (t < t_end - 1e-9 * dt) {
    std::swap(h, hp);  // hp = the state before the step
    apply_batch(p, 0, dz.as<double2>(), hp, n, y, n, B, false, "cn_apply");
    launch(ctx, "cn_vec", 48.0 * B * n, [&] {
      cn_rhs_kernel<<<g2, kT, 0, st>>>(n, B, y, dsrc.as<double>(), drates.as<double>(), v);
    });
    inner_solve(p, B, taus.data(), v, n, h, n, nullptr, rel.data());
    check_inner_cn(p, rel);
    const double t_prev = t;
    t += dt;
    ++steps;
    record(t_prev, hp, t, h);
  }
  if (mem != LT_MEM_DEVICE)
    LT_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * (size_t)B * n_samples * n, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  if (steps_out) *steps_out = steps;
}

void condition_estimate(lt_pencil p, double2 z, double* norm_a, double* norm_inv, double* cond) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  LT_REQUIRE(n >= 1, "estimate_norm_1: dimension must be positive");
  DeviceBuffer vec(sizeof(double2) * (size_t)n * 3, st);
  double2* x = vec.as<double2>();
  double2* y = x + n;
  double2* w = y + n;
  const unsigned gr = grid_for(n, ctx);
  DeviceBuffer part(sizeof(double) * gr + sizeof(int64_t) * gr, st);
  double* pd = part.as<double>();
  int64_t* pi = reinterpret_cast<int64_t*>(pd + gr);
  DeviceBuffer dz(sizeof(double2) * 2, st);
  const double2 zz[2] = {z, make_double2(z.x, -z.y)};
  LT_CUDA(cudaMemcpyAsync(dz.get(), zz, sizeof(zz), cudaMemcpyHostToDevice, st));
  std::vector<double> hd(gr);
  std::vector<int64_t> hi(gr);
  // the actions: forward / adjoint of A (kind 0) or of A^{-1} (kind 1)
  auto act = [&](int kind, bool adjoint, const double2* in, double2* outv) {
    if (kind == 0) {
      apply_batch(p, 0, dz.as<double2>() + (adjoint ? 1 : 0), in, n, outv, n, 1, false, "condest_apply");
      return;
    }
    std::vector<double> rel(1);
    const double2 tau = adjoint ? make_double2(z.x, -z.y) : z;
    inner_solve(p, 1, &tau, in, n, outv, n, nullptr, rel.data());
    if (!(rel[0] <= kInnerFloor * p->inner_tol))
      throw Error(LT_ERR_PRECONDITIONER, "estimate_condition_1norm: shift-and-invert solve failed to converge");
  };
  auto l1 = [&](const double2* v) {
    launch(ctx, "condest_vec", 16.0 * n, [&] { l1_partial_kernel<<<gr, kT, 0, st>>>(n, v, pd); });
    LT_CUDA(cudaMemcpyAsync(hd.data(), pd, sizeof(double) * gr, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    double s = 0.0;
    for (double d : hd) s += d;
    return s;
  };
  auto argmax = [&](const double2* v) {
    launch(ctx, "condest_vec", 16.0 * n, [&] { absmax_partial_kernel<<<gr, kT, 0, st>>>(n, v, pd, pi); });
    LT_CUDA(cudaMemcpyAsync(hd.data(), pd, sizeof(double) * gr, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaMemcpyAsync(hi.data(), pi, sizeof(int64_t) * gr, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    double best = -1.0;
    int64_t bi = 0;
    for (unsigned b = 0; b < gr; ++b)
      if (hi[b] >= 0 && (hd[b] > best || (hd[b] == best && hi[b] < bi))) { best = hd[b]; bi = hi[b]; }
    return bi;
  };
  // Hager's iteration (condest.cpp:11-41)
  auto norm1 = [&](int kind) {
    std::vector<double2> init(n, make_double2(1.0 / (double)n, 0.0));
    LT_CUDA(cudaMemcpyAsync(x, init.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    double best = 0.0;
    int64_t previous = -1;
    for (int iteration = 0; iteration < 6; ++iteration) {
      act(kind, false, x, y);
      const double estimate = l1(y);
      if (iteration > 0 && estimate <= best) break;
      best = std::max(best, estimate);
      launch(ctx, "condest_vec", 32.0 * n, [&] { sign_kernel<<<gr, kT, 0, st>>>(n, y, w); });
      act(kind, true, w, y);
      const int64_t pivot = argmax(y);
      if (pivot == previous) break;
      LT_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
      const double2 one = make_double2(1.0, 0.0);
      LT_CUDA(cudaMemcpyAsync(x + pivot, &one, sizeof(double2), cudaMemcpyHostToDevice, st));
      previous = pivot;
    }
    return best;
  };
  const double na = norm1(0);
  const double ni = norm1(1);
  if (norm_a) *norm_a = na;
  if (norm_inv) *norm_inv = ni;
  if (cond) *cond = na * ni;
}

}  // namespace lt
