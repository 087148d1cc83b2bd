// Dev probe: does the 512^3 K4 slowdown come from the direction-major layout
// (19 read + 19 write streams, each one direction array = 512 MB apart)?
// A pull-stream kernel with K4's access pattern (19 shifted loads, 19 stores,
// persistent grid, one plane per work item) over two layouts of the same
// 512x512xNZ fp32 state:
//   dir-major   : f[i*stride + x + nx*(y + ny*z)]            (current)
//   plane-inter : f[(z*19 + i)*plane + x + nx*y]              (19 planes of z together)
// Prints GB/s (152 B per cell update) for several NZ.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe_layout probe_layout.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ int cex[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
__constant__ int cey[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
__constant__ int cez[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};

struct P {
  const float* a[19];
  float* b[19];
};

// dstride: elements between directions; zstride: elements between z planes
__global__ void __launch_bounds__(128, 6) k_pull(P p, int nx, int ny, int nz, long long dstride,
                                                  long long zstride) {
  const int tx_n = nx / 128, ty_n = ny;  // K4's block shape: 128 cells of one row
  const int ncol = tx_n * ty_n;
  const int nitem = ncol * (nz - 2);
  for (int it = blockIdx.x; it < nitem; it += gridDim.x) {
    const int col = it % ncol, z = 1 + it / ncol;
    const int x = (col % tx_n) * 128 + threadIdx.x;
    const int y = col / tx_n;
    if (y == 0 || y == ny - 1 || x == 0 || x == nx - 1) continue;
    const long long m = x + (long long)nx * y + zstride * z;
    float s[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) s[i] = __ldg(p.a[i] + m);
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 19; ++i) t += s[i];
    t *= 1.0f / 19.0f;
#pragma unroll
    for (int i = 0; i < 19; ++i) p.b[i][m] = 0.9f * s[i] + 0.1f * t;
  }
}

// y-tiled: f[((z*nyt + y/TY)*19 + i)*(nx*TY) + x + nx*(y%TY)] -- the 19
// direction sub-arrays of a (z, y-tile) group lie within 19*nx*TY*4 bytes
// (TY = 8 at nx = 512: 304 KB) instead of 19 planes (19 MB) apart.
template <int LT>
__global__ void __launch_bounds__(128, 6) k_pull_tiled(const float* __restrict__ A, float* __restrict__ B,
                                                        int nx, int lnx, int ny, int nz) {
  constexpr int TY = 1 << LT;
  const int tx_n = nx / 128, ty_n = ny;
  const int ncol = tx_n * ty_n, nyt = ny >> LT;
  const long long tileN = (long long)nx << LT;
  const int nitem = ncol * (nz - 2);
  for (int it = blockIdx.x; it < nitem; it += gridDim.x) {
    const int col = it % ncol, z = 1 + it / ncol;
    const int x = (col % tx_n) * 128 + threadIdx.x;
    const int y = col / tx_n;
    if (y == 0 || y == ny - 1 || x == 0 || x == nx - 1) continue;
    float s[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) {
      const int xs = x - cex[i], ys = y - cey[i], zs = z - cez[i];
      const long long a = (((long long)zs * nyt + (ys >> LT)) * 19 + i) * tileN + xs + ((ys & (TY - 1)) << lnx);
      s[i] = __ldg(A + a);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 19; ++i) t += s[i];
    t *= 1.0f / 19.0f;
    const long long o = (((long long)z * nyt + (y >> LT)) * 19) * tileN + x + ((y & (TY - 1)) << lnx);
#pragma unroll
    for (int i = 0; i < 19; ++i) B[o + i * tileN] = 0.9f * s[i] + 0.1f * t;
  }
}

template <int LT>
void run_tiled(float* A, float* B, int nx, int ny, int nz, int nsm) {
  const int grid = nsm * 6;
  for (int w = 0; w < 3; ++w) k_pull_tiled<LT><<<grid, 128>>>(w & 1 ? B : A, w & 1 ? A : B, nx, 9, ny, nz);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = nz >= 256 ? 10 : 40;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_pull_tiled<LT><<<grid, 128>>>(r & 1 ? B : A, r & 1 ? A : B, nx, 9, ny, nz);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)(nx - 2) * (ny - 2) * (nz - 2);
  const double sec = ms / 1e3 / reps;
  printf("nz=%4d            y-tiled TY=%-3d %.3f ms  %.1f GLUPS  %.0f GB/s\n", nz, 1 << LT, sec * 1e3,
         cells / sec / 1e9, cells * 152 / sec / 1e9);
}

int main() {
  const int nx = 512, ny = 512;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int nz : {32, 128, 256, 512}) {
    const long long plane = (long long)nx * ny, n = plane * nz;
    float *A, *B;
    if (cudaMalloc(&A, 19 * n * 4) || cudaMalloc(&B, 19 * n * 4)) {
      printf("alloc failed nz=%d\n", nz);
      return 1;
    }
    cudaMemset(A, 0, 19 * n * 4);
    cudaMemset(B, 0, 19 * n * 4);
    for (int layout = 0; layout < 2; ++layout) {
      const long long dstride = layout == 0 ? n : plane;
      const long long zstride = layout == 0 ? plane : 19 * plane;
      P pa, pb;
      int ex[19], ey[19], ez[19];
      cudaMemcpyFromSymbol(ex, cex, sizeof ex);
      cudaMemcpyFromSymbol(ey, cey, sizeof ey);
      cudaMemcpyFromSymbol(ez, cez, sizeof ez);
      for (int i = 0; i < 19; ++i) {
        const long long src = -(ex[i] + (long long)nx * ey[i] + zstride * ez[i]);
        pa.a[i] = A + i * dstride + src;
        pa.b[i] = B + i * dstride;
        pb.a[i] = B + i * dstride + src;
        pb.b[i] = A + i * dstride;
      }
      const int grid = nsm * 6;
      for (int w = 0; w < 3; ++w) k_pull<<<grid, 128>>>(w & 1 ? pb : pa, nx, ny, nz, dstride, zstride);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = nz >= 256 ? 10 : 40;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) k_pull<<<grid, 128>>>(r & 1 ? pb : pa, nx, ny, nz, dstride, zstride);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double cells = (double)(nx - 2) * (ny - 2) * (nz - 2);
      const double s = ms / 1e3 / reps;
      printf("nz=%4d state %.1f GB  %-11s  %.3f ms  %.1f GLUPS  %.0f GB/s\n", nz, 2.0 * 19 * n * 4 / 1e9,
             layout == 0 ? "dir-major" : "plane-inter", s * 1e3, cells / s / 1e9, cells * 152 / s / 1e9);
    }
    if (nx == 512) {  // (lnx = 9 hard-wired)
      run_tiled<2>(A, B, nx, ny, nz, nsm);
      run_tiled<3>(A, B, nx, ny, nz, nsm);
      run_tiled<4>(A, B, nx, ny, nz, nsm);
    }
    cudaFree(A);
    cudaFree(B);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
