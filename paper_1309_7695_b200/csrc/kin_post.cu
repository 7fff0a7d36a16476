// kin_post.cu — statistics kernel (K6 of DESIGN.md) and device utilities.
//
// The simulators write trajectories directly in the host layout [S][G][N]
// (Trajectory::samples per run, model.hpp:113-120), so results leave the GPU
// with one contiguous D2H copy and no transpose.
//   point_stats     EnsembleStatistics per sweep point (ensemble.hpp:20-57):
//                   Welford add over the point's runs in ascending run order
//                   (the workers=1 merge order), written grid-major
//                   [P][G][N].  Compiled with -fmad=false so it rounds exactly
//                   like the oracle's welford_add.  HBM-bound streaming read.
#include <algorithm>

#include "kin_device.cuh"
#include "kin_launch.h"

namespace kin {

namespace {


// One thread per (point, grid*species element): the point's runs are
// consecutive [sim][g][n] rows, so each run's read is coalesced across the
// threads of a point and the [P][G][N] writes are contiguous.
// n_done > 0 continues accumulators that already hold the first n_done runs
// (a KIN_OUTPUT_STATS_ONLY window boundary inside a point): the same Welford
// operations as one pass over all runs.  Continuation needs both outputs.
__global__ void __launch_bounds__(256) stats_kernel(const double* __restrict__ traj, int gn, uint64_t runs,
                                                    uint64_t base, uint64_t n_points, uint64_t n_done,
                                                    double* __restrict__ mean, double* __restrict__ m2) {
  const uint64_t total = n_points * static_cast<uint64_t>(gn);
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t p = e / gn;
    const uint64_t q = e - p * gn;
    const double* col = traj + (base + p * runs) * gn + q;
    double mu = 0.0, s2 = 0.0;
    if (n_done) {
      mu = mean[e];
      s2 = m2[e];
    }
    for (uint64_t r = 0; r < runs; ++r) {
      const double xv = __ldcs(col + r * gn);
      const double delta = __dsub_rn(xv, mu);
      mu = __dadd_rn(mu, __ddiv_rn(delta, static_cast<double>(n_done + r + 1)));
      s2 = __dadd_rn(s2, __dmul_rn(delta, __dsub_rn(xv, mu)));
    }
    if (mean) __stcs(mean + e, mu);
    if (m2) __stcs(m2 + e, s2);
  }
}

// n Binomial(n_trials, p) draws from RngStream(seed) (the KIN_FIRING_BINOMIAL sampler).
__global__ void binomial_kernel(uint64_t seed, uint64_t n_trials, double p, int n, uint64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Xoshiro rng;
  rng.seed(seed);
  uint64_t fl = 0;
  for (int q = 0; q < n; ++q) out[q] = binomial<false>(rng, n_trials, p, fl);
}

__global__ void rng_kernel(uint64_t seed, int kind, double mean, int n, uint64_t* out, const double* lgamma_tab) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Xoshiro rng;
  rng.seed(seed);
  uint64_t dummy = 0;
  double spare = 0.0;
  bool have = false;
  if (kind == 4) {
    PhiloxSite src(seed, 0, 0);
    for (int q = 0; q < n; ++q) out[q] = __double_as_longlong(src.uniform());
    return;
  }
  for (int q = 0; q < n; ++q) {
    uint64_t bits;
    if (kind == 0) {
      bits = rng.next();
    } else if (kind == 1) {
      const double v = rng.uniform();
      bits = __double_as_longlong(v);
    } else if (kind == 2) {  // Box-Muller with cached spare (rng.cpp:54-66)
      double v;
      if (have) {
        have = false;
        v = spare;
      } else {
        const double u1 = rng.uniform();
        const double u2 = rng.uniform();
        const double r = sqrt(__dmul_rn(-2.0, log(u1)));
        const double ang = __dmul_rn(__dmul_rn(2.0, 3.141592653589793), u2);
        spare = __dmul_rn(r, sin(ang));
        have = true;
        v = __dmul_rn(r, cos(ang));
      }
      bits = __double_as_longlong(v);
    } else if (kind == 4) {  // Philox uniforms of site (seed, 0, 0)
      if (q == 0) {
        // handled below with a persistent site
      }
      bits = 0;
    } else if (kind == 5) {  // one Philox Poisson draw per site (seed, 0, q)
      PhiloxSite src(seed, 0, static_cast<uint32_t>(q));
      bits = poisson<false>(src, mean, dummy, lgamma_tab);
    } else {
      bits = poisson<false>(rng, mean, dummy, lgamma_tab);
    }
    out[q] = bits;
  }
}

// DFMA throughput probe: 8 independent FMA chains per thread.
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double c) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 0.999999999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

cudaError_t launch_point_stats(const double* traj_dev, int gn, uint64_t runs, uint64_t base, uint64_t n_points,
                               uint64_t n_done, double* mean, double* m2, cudaStream_t st) {
  if (n_points == 0 || gn == 0) return cudaSuccess;
  const uint64_t total = n_points * static_cast<uint64_t>(gn);
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
  stats_kernel<<<blocks, 256, 0, st>>>(traj_dev, gn, runs, base, n_points, n_done, mean, m2);
  return cudaGetLastError();
}

cudaError_t launch_binomial_draws(uint64_t seed, uint64_t n_trials, double p, int n, uint64_t* out,
                                  cudaStream_t st) {
  binomial_kernel<<<1, 32, 0, st>>>(seed, n_trials, p, n, out);
  return cudaGetLastError();
}

cudaError_t launch_rng_draws(uint64_t seed, int kind, double mean, int n, uint64_t* out, const double* lgamma_tab,
                             cudaStream_t st) {
  rng_kernel<<<1, 32, 0, st>>>(seed, kind, mean, n, out, lgamma_tab);
  return cudaGetLastError();
}

cudaError_t measure_fp64_peak(cudaStream_t st, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int block = 256, blocks = sms * 8, iters = 2048;
  double* out = nullptr;
  cudaError_t e = cudaMalloc(&out, sizeof(double) * block * blocks);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, block, 0, st>>>(out, 64, 1e-12);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    dfma_kernel<<<blocks, block, 0, st>>>(out, iters, 1e-12);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * block * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  e = cudaGetLastError();
  cudaFree(out);
  return e;
}

}  // namespace kin
