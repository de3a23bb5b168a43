// BP1.0 S3 line operator on FP64 tensor cores vs the kernel's folded DFMA form
// (verdict r1 "missing" item 4: a measured DMMA variant of the folded I / I^T
// halves).  Both variants apply, to every i-line x (n = 8 GLL values) of a
// shared-memory tile,  out = I^T ( w .* (I x) )  with I the 9 x 8 GLL -> GL
// interpolation matrix of N = 7 -- exactly hx_bp1.cu's S3 -- and write the
// result back in place; the tile is re-processed ITERS times so the timing
// is the shared-memory + FP64 work of the stage alone (no HBM).
//
//   dfma: one line per thread, fold_apply<9,8> / fold_apply<8,9> with the
//         coefficients as uniform constant-bank operands (hx_common.cuh)
//   dmma: eight lines per warp-group step, mma.sync.m8n8k4.f64:
//         Y (16 x 8) = I_pad (16 x 8) X (8 x 8 lines)  -> 2 m-tiles x 2 k-steps
//         Z = w .* Y in the accumulator layout, staged through shared memory
//         O (8 x 8) = I^T_pad (8 x 12) Z (12 x 8)      -> 3 k-steps
//         i.e. 7 DMMAs (1792 FMA slots) per 8 lines against 8 x 113 FP64
//         instructions (904 lane-ops) folded
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_s3_probe tools/dmma_s3_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

constexpr int n = 8, m = 9;
constexpr int LINES = 248;  // lines per CTA tile: 3 elements x 81 i-lines, rounded up to 8
constexpr int ITERS = 200;
constexpr int LS = n + 1;  // line stride in shared memory (odd: conflict-free one-line-per-thread access)

struct Coef {
  double I[m * n];   // row-major 9 x 8
  double e[5][5];    // folded I: even part rows 0..4 (cols 0..3 + middle unused for n even)
  double o[5][4];
  double te[4][5];   // folded I^T (8 x 9): even part, col 4 = middle input
  double to[4][4];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// --- DFMA folded form (one line per thread) --------------------------------
__global__ void __launch_bounds__(256) s3_dfma(double* g, const double* gw,
                                               const __grid_constant__ Coef c) {
  __shared__ double tile[LINES * LS];
  __shared__ double wt[LINES * m];
  for (int i = threadIdx.x; i < LINES * n; i += blockDim.x) tile[i / n * LS + i % n] = g[blockIdx.x * LINES * n + i];
  for (int i = threadIdx.x; i < LINES * m; i += blockDim.x) wt[i] = gw[i];
  __syncthreads();
  for (int it = 0; it < ITERS; ++it) {
    for (int ln = threadIdx.x; ln < LINES; ln += blockDim.x) {
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = tile[ln * LS + t];
      double xe[4], xo[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) { xe[b] = x[b] + x[7 - b]; xo[b] = x[b] - x[7 - b]; }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double ye = c.e[a][0] * xe[0], yo = c.o[a][0] * xo[0];
#pragma unroll
        for (int b = 1; b < 4; ++b) { ye = fma(c.e[a][b], xe[b], ye); yo = fma(c.o[a][b], xo[b], yo); }
        y[a] = ye + yo;
        y[8 - a] = ye - yo;
      }
      {
        double ye = c.e[4][0] * xe[0];
#pragma unroll
        for (int b = 1; b < 4; ++b) ye = fma(c.e[4][b], xe[b], ye);
        y[4] = ye;
      }
#pragma unroll
      for (int a = 0; a < m; ++a) y[a] *= wt[ln * m + a];
      double ze[4], zo[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) { ze[b] = y[b] + y[8 - b]; zo[b] = y[b] - y[8 - b]; }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double ve = c.te[a][0] * ze[0], vo = c.to[a][0] * zo[0];
#pragma unroll
        for (int b = 1; b < 4; ++b) { ve = fma(c.te[a][b], ze[b], ve); vo = fma(c.to[a][b], zo[b], vo); }
        ve = fma(c.te[a][4], y[4], ve);
        x[a] = ve + vo;
        x[7 - a] = ve - vo;
      }
#pragma unroll
      for (int t = 0; t < n; ++t) tile[ln * LS + t] = x[t];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < LINES * n; i += blockDim.x) g[blockIdx.x * LINES * n + i] = tile[i / n * LS + i % n];
}

// --- DMMA form (eight lines per warp step) ---------------------------------
__global__ void __launch_bounds__(256) s3_dmma(double* g, const double* gw,
                                               const __grid_constant__ Coef c) {
  __shared__ double tile[LINES * LS];
  __shared__ double wt[LINES * m];
  __shared__ double zs[8][12 * 8 + 4];  // per warp: Z (12 x 8 lines), row-major, padded
  for (int i = threadIdx.x; i < LINES * n; i += blockDim.x) tile[i / n * LS + i % n] = g[blockIdx.x * LINES * n + i];
  for (int i = threadIdx.x; i < LINES * m; i += blockDim.x) wt[i] = gw[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  // A fragments: I_pad rows 8*mt + r, cols 4*ks + q (rows >= 9 are zero)
  double aI[2][2], aT[3];
  for (int mt = 0; mt < 2; ++mt)
    for (int ks = 0; ks < 2; ++ks) {
      const int row = 8 * mt + r, col = 4 * ks + q;
      aI[mt][ks] = row < m ? c.I[row * n + col] : 0.0;
    }
  // I^T_pad (8 x 12): row r, cols 4*ks + q (cols >= 9 are zero)
  for (int ks = 0; ks < 3; ++ks) {
    const int col = 4 * ks + q;
    aT[ks] = col < m ? c.I[col * n + r] : 0.0;
  }
  double* z = zs[warp];
  for (int i = lane; i < 12 * 8 + 4; i += 32) z[i] = 0.0;
  __syncthreads();
  for (int it = 0; it < ITERS; ++it) {
    for (int l0 = warp * 8; l0 < LINES; l0 += 8 * 8) {
      // Y = I X: B fragment = X[k = 4ks + q][line = r]
      double y[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double b = tile[(l0 + r) * LS + 4 * ks + q];
        dmma(y[0][0], y[0][1], aI[0][ks], b);
        dmma(y[1][0], y[1][1], aI[1][ks], b);
      }
      // scale in the accumulator layout: Y[row = 8 mt + r][line = 2q + j]
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int row = 8 * mt + r, line = 2 * q + j;
          if (row < m) z[row * 8 + line] = y[mt][j] * wt[(l0 + line) * m + row];
        }
      __syncwarp();
      // O = I^T Z: B fragment = Z[k = 4ks + q][line = r]
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) dmma(o0, o1, aT[ks], z[(4 * ks + q) * 8 + r]);
      __syncwarp();
      // O[i = r][line = 2q + j] back into the line
      tile[(l0 + 2 * q) * LS + r] = o0;
      tile[(l0 + 2 * q + 1) * LS + r] = o1;
      __syncwarp();
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < LINES * n; i += blockDim.x) g[blockIdx.x * LINES * n + i] = tile[i / n * LS + i % n];
}

// GLL / GL nodes of N = 7 and the barycentric interpolation matrix
static void nodes(std::vector<double>& x, int p, bool lobatto) {
  x.assign(p, 0.0);
  for (int i = 0; i < p; ++i) {
    double t = -std::cos(M_PI * (lobatto ? double(i) / (p - 1) : (i + 0.75) / (p + 0.5)));
    for (int k = 0; k < 100; ++k) {  // Newton on P_{p-1}' (Lobatto) or P_p (Gauss)
      const int d = lobatto ? p - 1 : p;
      double p0 = 1, p1 = t, dp = 1;
      for (int j = 2; j <= d; ++j) {
        const double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      dp = d * (t * p1 - p0) / (t * t - 1);
      if (lobatto) {
        if (i == 0 || i == p - 1) break;
        const double d2 = (2 * t * dp - d * (d + 1) * p1) / (1 - t * t);
        const double dt = dp / d2;
        t -= dt;
        if (std::fabs(dt) < 1e-15) break;
      } else {
        const double dt = p1 / dp;
        t -= dt;
        if (std::fabs(dt) < 1e-15) break;
      }
    }
    x[i] = t;
  }
}

int main() {
  std::vector<double> xg, xq;
  nodes(xg, n, true);
  nodes(xq, m, false);
  Coef c{};
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < n; ++b) {
      double l = 1;
      for (int k = 0; k < n; ++k)
        if (k != b) l *= (xq[a] - xg[k]) / (xg[b] - xg[k]);
      c.I[a * n + b] = l;
    }
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b < 4; ++b) {
      c.e[a][b] = 0.5 * (c.I[a * n + b] + c.I[a * n + 7 - b]);
      c.o[a][b] = a < 4 ? 0.5 * (c.I[a * n + b] - c.I[a * n + 7 - b]) : 0.0;
    }
  for (int a = 0; a < 4; ++a) {  // I^T (8 x 9)
    for (int b = 0; b < 4; ++b) {
      c.te[a][b] = 0.5 * (c.I[b * n + a] + c.I[(8 - b) * n + a]);
      c.to[a][b] = 0.5 * (c.I[b * n + a] - c.I[(8 - b) * n + a]);
    }
    c.te[a][4] = c.I[4 * n + a];
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4;
  const size_t nd = size_t(blocks) * LINES * n;
  std::vector<double> h(nd), w(LINES * m);
  srand(1);
  for (auto& v : h) v = rand() / double(RAND_MAX) - 0.5;
  // scale w by 1 / lambda_max(I^T I) so ITERS passes neither blow up nor
  // underflow (power iteration on the 8 x 8 normal matrix)
  double lam = 0;
  {
    std::vector<double> v(n, 1.0), u(n);
    for (int itp = 0; itp < 200; ++itp) {
      std::vector<double> t(m, 0.0);
      for (int a = 0; a < m; ++a)
        for (int b = 0; b < n; ++b) t[a] += c.I[a * n + b] * v[b];
      for (int b = 0; b < n; ++b) {
        u[b] = 0;
        for (int a = 0; a < m; ++a) u[b] += c.I[a * n + b] * t[a];
      }
      double nn = 0;
      for (double x : u) nn += x * x;
      nn = std::sqrt(nn);
      lam = nn;
      for (int b = 0; b < n; ++b) v[b] = u[b] / nn;
    }
  }
  for (auto& v : w) v = (0.999 + 0.001 * rand() / double(RAND_MAX)) / lam;
  double *d1, *d2, *dw;
  cudaMalloc(&d1, nd * 8);
  cudaMalloc(&d2, nd * 8);
  cudaMalloc(&dw, w.size() * 8);
  cudaMemcpy(dw, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto k, double* d) {
    cudaMemcpy(d, h.data(), nd * 8, cudaMemcpyHostToDevice);
    k<<<blocks, 256>>>(d, dw, c);  // warm-up
    cudaMemcpy(d, h.data(), nd * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k<<<blocks, 256>>>(d, dw, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double lines = double(blocks) * LINES * ITERS;
    printf("%-5s %8.3f ms  %7.3f ns per 1000 lines per SM  (%.2f Glines/s)\n", name, ms,
           ms * 1e6 / lines * sms * 1000, lines / (ms * 1e-3) / 1e9);
  };
  run("dfma", s3_dfma, d1);
  run("dmma", s3_dmma, d2);
  std::vector<double> r1(nd), r2(nd);
  cudaMemcpy(r1.data(), d1, nd * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), d2, nd * 8, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (size_t i = 0; i < nd; ++i) {
    num += (r1[i] - r2[i]) * (r1[i] - r2[i]);
    den += r1[i] * r1[i];
  }
  printf("rel L2 dmma vs dfma after %d passes: %.3e   status: %s, SMs %d\n", ITERS,
         std::sqrt(num / (den > 0 ? den : 1)), cudaGetErrorString(cudaGetLastError()), sms);
  return 0;
}
