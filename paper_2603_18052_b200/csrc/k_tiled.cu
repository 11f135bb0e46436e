// k_tiled.cu — K1c: shared-P propagation for any n with P streamed from L2
// (config 3: d = 27, n = 729, P = 8.5 MB, 1,024 trajectories, 200 steps), and
// the plain batched complex GEMM used by the GPU expm.
//
// One step is a complex GEMM  V_next (n x B) = P (n x n) * V (n x B).  P and both
// state buffers (2 x 12 MB at config 3) stay L2-resident (126 MB L2), so the
// bound is the DMMA pipe. The kernel is PERSISTENT (cooperative launch, all
// CTAs co-resident): per step every CTA pulls 32x32 complex output tiles from
// an atomic counter (dynamic balance: 736 tiles on 148 SMs), computes each tile
// with a 3-stage cp.async pipeline feeding m8n8k4 DMMAs in real form
// (common.cuh), writes it to the other state buffer, and all CTAs meet at a
// grid barrier before the next step (every output row needs every input row).
//
// Tile geometry: 32 complex rows (64 real, 8 m-tiles) x 32 columns (4 n-tiles),
// K chunk 16 complex (8 k-steps); 8 warps, each 2 m-tiles x 2 n-tiles.
// Shared strides SA = 2 (mod 8), SB = 4 (mod 8) complex make every fragment
// load bank-conflict free.
//
// Replaces step_soa_kernel (proj/src/kernels_variants.cpp:26-41) inside
// evolve (proj/src/propagate.cpp:85-92), batched; the GEMM replaces
// lb::matmul (proj/src/complex_matrix.cpp:30-56) inside expm.
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {

namespace {

constexpr int BM = 32, BN = 32, BK = 16, STAGES = 3, THREADS = 256;
constexpr int SA = 18, SB = 36;  // complex strides (see header)
constexpr int A_ELEMS = BM * SA, B_ELEMS = BK * SB;
constexpr size_t kSmemBytes = size_t(STAGES) * (A_ELEMS + B_ELEMS) * sizeof(double2);

struct TileCtx {
  int tid, lane, wm, wn;
  AFragLane af;
  __device__ TileCtx() : tid(threadIdx.x), lane(threadIdx.x & 31), wm((threadIdx.x >> 5) >> 1),
                         wn((threadIdx.x >> 5) & 1), af(threadIdx.x & 31) {}
};

__device__ __forceinline__ void load_stage(double2* as, double2* bs, const double2* __restrict__ A,
                                           long long lda, const double2* __restrict__ B,
                                           long long ldb, int M, int N, int K, int m0, int n0,
                                           int k0, int tid) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = tid + r * THREADS;
    {  // A: 32 rows x 16 complex
      const int row = e >> 4, col = e & 15;
      const bool ok = (m0 + row < M) && (k0 + col < K);
      const double2* src = ok ? A + (long long)(m0 + row) * lda + (k0 + col) : A;
      cp_async16(as + row * SA + col, src, ok);
    }
    {  // B: 16 rows x 32 complex
      const int row = e >> 5, col = e & 31;
      const bool ok = (k0 + row < K) && (n0 + col < N);
      const double2* src = ok ? B + (long long)(k0 + row) * ldb + (n0 + col) : B;
      cp_async16(bs + row * SB + col, src, ok);
    }
  }
}

// acc[mi][ni][2] += A(m0.., :) * B(:, n0..) over the full K.
__device__ __forceinline__ void gemm_tile(const double2* __restrict__ A, long long lda,
                                          const double2* __restrict__ B, long long ldb, int M,
                                          int N, int K, int m0, int n0, double (&acc)[2][2][2],
                                          double2* smem, const TileCtx& c) {
  double2* as = smem;
  double2* bs = smem + STAGES * A_ELEMS;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const int nk = (K + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load_stage(as + st * A_ELEMS, bs + st * B_ELEMS, A, lda, B, ldb, M, N, K, m0, n0, st * BK, c.tid);
    cp_async_commit();
  }
  // per-lane fragment offsets (doubles) inside a stage
  const int a_off = 2 * ((c.wm * 2 * 4 + c.af.di) * SA + c.af.dj) + c.af.comp;
  const int b_off = 2 * (((c.lane & 3) >> 1) * SB + c.wn * 2 * 8 + (c.lane >> 2)) + (c.lane & 1);
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kc + STAGES - 1;
      if (nxt < nk)
        load_stage(as + (nxt % STAGES) * A_ELEMS, bs + (nxt % STAGES) * B_ELEMS, A, lda, B, ldb, M,
                   N, K, m0, n0, nxt * BK, c.tid);
      cp_async_commit();
    }
    const double* ad = reinterpret_cast<const double*>(as + (kc % STAGES) * A_ELEMS) + a_off;
    const double* bd = reinterpret_cast<const double*>(bs + (kc % STAGES) * B_ELEMS) + b_off;
#pragma unroll
    for (int ks = 0; ks < BK / 2; ++ks) {
      double a[2], b[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[mi] = c.af.sign(ad[2 * (mi * 4 * SA) + 4 * ks]);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = bd[2 * (2 * ks * SB + ni * 8)];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // stages free for the next tile
}

__device__ __forceinline__ void store_tile(double2* __restrict__ C, long long ldc, int M, int N,
                                           int m0, int n0, const double (&acc)[2][2][2],
                                           const TileCtx& c) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      int coff;
      const double2 z = pair_complex(acc[mi][ni], c.lane, coff);
      const int i = m0 + (c.wm * 2 + mi) * 4 + (c.lane >> 3);
      const int col = n0 + (c.wn * 2 + ni) * 8 + coff;
      if (i < M && col < N) C[(long long)i * ldc + col] = z;
    }
}

// ---- plain batched GEMM (expm) --------------------------------------------
__global__ void __launch_bounds__(THREADS) zgemm_kernel(const double2* __restrict__ A,
                                                        const double2* __restrict__ B,
                                                        double2* __restrict__ C, int n,
                                                        long long sa, long long sb, long long sc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const TileCtx c;
  const int b = blockIdx.z;
  double acc[2][2][2];
  gemm_tile(A + b * sa, n, B + b * sb, n, n, n, n, blockIdx.x * BM, blockIdx.y * BN, acc,
            reinterpret_cast<double2*>(smem_raw), c);
  store_tile(C + b * sc, n, n, n, blockIdx.x * BM, blockIdx.y * BN, acc, c);
}

// ---- persistent stepping ----------------------------------------------------
struct StepCtl {
  unsigned int tile_ctr[2];
  unsigned int barrier;
  unsigned int pad;
};

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(THREADS) tiled_evolve_kernel(const double2* __restrict__ P, int n,
                                                               double2* v0, double2* v1,
                                                               int batch, int64_t steps,
                                                               StepCtl* ctl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_tile;
  const TileCtx c;
  const int tiles_m = (n + BM - 1) / BM, tiles_n = (batch + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  double2* cur = v0;
  double2* nxt = v1;
  for (int64_t s = 0; s < steps; ++s) {
    const int par = int(s & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->tile_ctr[par ^ 1] = 0u;  // next step's counter
    while (true) {
      if (threadIdx.x == 0) s_tile = int(atomicAdd(&ctl->tile_ctr[par], 1u));
      __syncthreads();
      const int t = s_tile;
      __syncthreads();
      if (t >= ntiles) break;
      // column-major tile order: consecutive CTAs share the same V columns
      const int tm = t % tiles_m, tn = t / tiles_m;
      double acc[2][2][2];
      gemm_tile(P, n, cur, batch, n, batch, n, tm * BM, tn * BN, acc,
                reinterpret_cast<double2*>(smem_raw), c);
      store_tile(nxt, batch, n, batch, tm * BM, tn * BN, acc, c);
    }
    grid_barrier(&ctl->barrier, unsigned(s + 1) * gridDim.x);
    double2* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

// layout conversion between the user's [b][k] (SoA / AoS) and V[k][b] (AoS)
template <Layout L, bool ToV>
__global__ void convert_kernel(double* x_re, double* x_im, double* x_aos, double2* v, int n,
                               int batch) {
  __shared__ double2 tile[32][33];
  const int kb = blockIdx.x * 32, bb = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (ToV) {
    for (int r = ty; r < 32; r += 8) {  // read x[b = bb + r][k = kb + tx]
      const int b = bb + r, k = kb + tx;
      double2 z = make_double2(0.0, 0.0);
      if (b < batch && k < n) {
        if (L == Layout::soa)
          z = make_double2(x_re[(long long)b * n + k], x_im[(long long)b * n + k]);
        else
          z = reinterpret_cast<const double2*>(x_aos)[(long long)b * n + k];
      }
      tile[r][tx] = z;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // write v[k = kb + r][b = bb + tx]
      const int k = kb + r, b = bb + tx;
      if (k < n && b < batch) v[(long long)k * batch + b] = tile[tx][r];
    }
  } else {
    for (int r = ty; r < 32; r += 8) {  // read v[k = kb + r][b = bb + tx]
      const int k = kb + r, b = bb + tx;
      tile[r][tx] = (k < n && b < batch) ? v[(long long)k * batch + b] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // write x[b = bb + r][k = kb + tx]
      const int b = bb + r, k = kb + tx;
      if (b < batch && k < n) {
        const double2 z = tile[tx][r];
        if (L == Layout::soa) {
          x_re[(long long)b * n + k] = z.x;
          x_im[(long long)b * n + k] = z.y;
        } else {
          reinterpret_cast<double2*>(x_aos)[(long long)b * n + k] = z;
        }
      }
    }
  }
}

template <bool ToV>
void convert(double* x_re, double* x_im, double* x_aos, double2* v, int n, int batch,
             Layout layout, cudaStream_t s) {
  const dim3 grid((n + 31) / 32, (batch + 31) / 32), block(32, 8);
  if (layout == Layout::soa)
    convert_kernel<Layout::soa, ToV><<<grid, block, 0, s>>>(x_re, x_im, x_aos, v, n, batch);
  else
    convert_kernel<Layout::aos, ToV><<<grid, block, 0, s>>>(x_re, x_im, x_aos, v, n, batch);
  LBG_CHECK_LAUNCH("convert_kernel");
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

int sm_count() {
  static int count = [] {
    int dev = 0, c = 0;
    check_cuda(cudaGetDevice(&dev), "get device");
    check_cuda(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev), "sm count");
    return c;
  }();
  return count;
}

size_t tiled_workspace(size_t n, int64_t batch) {
  return 2 * align_up(sizeof(double2) * n * size_t(batch)) + align_up(sizeof(StepCtl));
}

void launch_tiled_evolve(const double* p_dev, size_t n, double* x_re, double* x_im, double* x_aos,
                         int64_t batch, int64_t steps, Layout layout, void* work, cudaStream_t s) {
  if (batch <= 0) return;
  if (batch > (1ll << 30) || n > (1u << 20)) throw invalid_argument("tiled: shape too large");
  if (!work) throw invalid_argument("tiled: workspace required");
  char* w = static_cast<char*>(work);
  double2* v0 = reinterpret_cast<double2*>(w);
  double2* v1 = reinterpret_cast<double2*>(w + align_up(sizeof(double2) * n * size_t(batch)));
  StepCtl* ctl = reinterpret_cast<StepCtl*>(w + 2 * align_up(sizeof(double2) * n * size_t(batch)));
  const int ni = int(n), bi = int(batch);
  convert<true>(x_re, x_im, x_aos, v0, ni, bi, layout, s);
  check_cuda(cudaMemsetAsync(ctl, 0, sizeof(StepCtl), s), "memset ctl");

  static int occ = [] {
    check_cuda(cudaFuncSetAttribute(tiled_evolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmemBytes)),
               "smem attr");
    int o = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tiled_evolve_kernel, THREADS, kSmemBytes),
               "occupancy");
    return o;
  }();
  const int ntiles = ((ni + BM - 1) / BM) * ((bi + BN - 1) / BN);
  int grid = std::min(occ * sm_count(), ntiles);
  if (grid < 1) grid = 1;
  const double2* p2 = reinterpret_cast<const double2*>(p_dev);
  int64_t st = steps;
  void* args[] = {(void*)&p2, (void*)&ni, (void*)&v0, (void*)&v1, (void*)&bi, (void*)&st, (void*)&ctl};
  if (steps > 0) {
    check_cuda(cudaLaunchCooperativeKernel((const void*)tiled_evolve_kernel, dim3(grid), dim3(THREADS),
                                           args, kSmemBytes, s),
               "tiled_evolve_kernel (cooperative)");
    note_launch();
  }
  convert<false>(x_re, x_im, x_aos, (steps & 1) ? v1 : v0, ni, bi, layout, s);
}

void launch_zgemm(const double* a, const double* b, double* c, int n, int batch, long long stride_a,
                  long long stride_b, long long stride_c, cudaStream_t s) {
  static bool init = [] {
    check_cuda(cudaFuncSetAttribute(zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmemBytes)),
               "smem attr");
    return true;
  }();
  (void)init;
  const dim3 grid((n + BM - 1) / BM, (n + BN - 1) / BN, batch);
  zgemm_kernel<<<grid, THREADS, kSmemBytes, s>>>(reinterpret_cast<const double2*>(a),
                                                 reinterpret_cast<const double2*>(b),
                                                 reinterpret_cast<double2*>(c), n, stride_a, stride_b,
                                                 stride_c);
  LBG_CHECK_LAUNCH("zgemm_kernel");
}

}  // namespace lbg
