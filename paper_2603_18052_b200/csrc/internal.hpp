// internal.hpp — host-side launchers shared between the kernel translation
// units and the C-ABI layer (capi.cu). Not part of the public boundary.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace lbg {

// error types mirror the reference's exception classes (mapped to LBG_* codes)
struct invalid_argument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct runtime_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void note_launch(int n = 1);  // launch counter (capi.cu)
void launch_scale(double* x, std::size_t n, double s, cudaStream_t st);  // x *= s (capi.cu)

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}
#define LBG_CHECK_LAUNCH(what)                  \
  do {                                          \
    ::lbg::note_launch();                       \
    ::lbg::check_cuda(cudaGetLastError(), what); \
  } while (0)

enum class Layout { soa, aos };

// K1a — n == 9, P in the constant bank (kernel parameter), DFMA (k_dfma9.cu)
void launch_dfma9(const double* p_aos_host_or_null, const double* p_dev, double* x_re,
                  double* x_im, double* x_aos, int64_t batch, int64_t steps, Layout layout,
                  cudaStream_t s);
// K2 — one warp per trajectory chain, latency-bound (k_chain.cu)
bool chain_supported(std::size_t n);
void launch_chain(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos,
                  int64_t batch, int64_t steps, Layout layout, cudaStream_t s);
// GRAPE chain over all segments in one launch, one trajectory (k_chain.cu)
void launch_chain_segments(const double* props, std::size_t n, int64_t segments, int64_t sps,
                           double* x_aos, cudaStream_t s);
// K1b — n <= 84, P resident in shared memory, DMMA (k_smem.cu)
bool smem_supported(std::size_t n);
void launch_smem(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos,
                 int64_t batch, int64_t steps, Layout layout, cudaStream_t s);
// K1b-C — n = 81 on 2-CTA clusters, DSMEM exchange of a split n-tile (k_cluster.cu)
bool cluster_supported(std::size_t n);
bool cluster_preferred(std::size_t n, int64_t batch);
int64_t cluster_cost(std::size_t n, int64_t batch);  // DMMA slots per sub-partition per step
int64_t smem81_cost(int64_t batch);
// K1b-K — n = 81 at small batches: 2-CTA clusters split K, P in registers (k_ksplit.cu)
bool ksplit_supported(std::size_t n);
int ksplit_group(std::size_t n, int64_t batch);
int64_t ksplit_cost(std::size_t n, int64_t batch);
void launch_ksplit(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos, int64_t batch,
                   int64_t steps, Layout layout, cudaStream_t s);
void launch_smem_cluster(const double* p_dev, double* x_re, double* x_im, double* x_aos, int64_t batch,
                         int64_t steps, Layout layout, cudaStream_t s);
// K1c — any n, persistent DMMA tiles streamed from L2 (k_tiled.cu)
std::size_t tiled_workspace(std::size_t n, int64_t batch);
void launch_tiled_evolve(const double* p_dev, std::size_t n, double* x_re, double* x_im,
                         double* x_aos, int64_t batch, int64_t steps, Layout layout, void* work,
                         cudaStream_t s);
// K1c-R — the same engine on real matrices (density mode beyond n = 84)
std::size_t tiled_real_workspace(std::size_t n, int64_t batch);
void launch_tiled_evolve_real(const double* p_dev, std::size_t n, double* x, int64_t batch, int64_t steps,
                              void* work, cudaStream_t s);
// K2b / K2c — latency kernels for one or a few trajectories (k_single.cu)
bool cta_chain_supported(std::size_t n);
void launch_cta_chain(const double* p, std::size_t n, double* x_aos, int64_t batch, int64_t steps,
                      cudaStream_t s);
void launch_cta_chain_segments(const double* props, std::size_t n, int64_t segments, int64_t sps,
                               double* x_aos, cudaStream_t s);
bool rowsplit_supported(std::size_t n, int64_t batch);
std::size_t rowsplit_workspace(std::size_t n, int64_t batch);
void launch_rowsplit(const double* p, std::size_t n, double* x_aos, int64_t batch, int64_t steps,
                     void* work, cudaStream_t s);
// automatic-choice AoS stepping (capi.cu)
void evolve_dev_aos(const double* p, std::size_t n, double* x_aos, int64_t batch, int64_t steps, void* work,
                    cudaStream_t s);
// density-matrix mode: shared P applied to the real coordinates (k_density.cu)
bool density_supported(std::size_t n);
bool density_uses_tile_engine(std::size_t n);  // n > 84: the cooperative real K1c
std::size_t density_workspace(std::size_t n, int64_t batch);
constexpr int kDensityHermitian = 0, kDensityGeneral = 1, kDensityAuto = 2;  // LBG_DENSITY_*
void launch_density(const double* p, std::size_t d, double* rho, int64_t batch, int64_t steps,
                    int mode, void* work, cudaStream_t s);
// plain batched complex GEMM C[b] = A[b] * B[b] (n x n, AoS), DMMA tiles;
// strides in complex elements
void launch_zgemm(const double* a, const double* b, double* c, int n, int batch,
                  long long stride_a, long long stride_b, long long stride_c, cudaStream_t s);
// the same engine on real matrices: leading dimension ld (even, >= n), strides 0 or n * ld doubles
// cond (device, optional): when cond_idx >= *cond the launch copies A into C instead
void launch_dgemm(const double* a, const double* b, double* c, int n, int ld, int batch, long long stride_a,
                  long long stride_b, long long stride_c, cudaStream_t s, const int* cond = nullptr,
                  int cond_idx = 0);

// model kernels (k_model.cu)
void launch_build_lindbladian(std::size_t d, const double* h, std::size_t n_ops,
                              const double* ops, double* out, cudaStream_t s);
constexpr std::size_t kExpmStreamN = 128;  // expm products on the stream-K engine from here
std::size_t expm_workspace(std::size_t n);  // bytes (lbg_expm_workspace)
// flag |= 1 when any of p[0 .. count) is not finite (k_validate.cu)
void launch_flag_nonfinite(const double* p, long long count, unsigned* flag, cudaStream_t s);
void launch_flag_nonhermitian(const double* m, long long d, unsigned* flag, cudaStream_t s);
// batched building blocks (k_model.cu)
void launch_build_lindbladian_batched(std::size_t d, const double* h, std::size_t n_ops, const double* ops,
                                      int64_t batch, double* out, cudaStream_t s);
std::size_t expm_batched_workspace(std::size_t n, int64_t batch);
void expm_batched_dev(const double* a, std::size_t n, int64_t batch, double dt, double* out, void* work,
                      cudaStream_t s);
// one complex GEMM C = A B (n x n) on the persistent stream-K engine (k_tiled.cu)
std::size_t zgemm_stream_workspace(int n);
void launch_zgemm_stream(const double* a, const double* b, double* c, int n, void* aux, cudaStream_t s);
void expm_dev(const double* a, std::size_t n, double dt, double* out, double* work,
              cudaStream_t s);
void launch_check_state(const double* x, std::size_t d, int64_t batch, double* out3,
                        cudaStream_t s);
void launch_planes_to_aos(const double* re, const double* im, long long count, double* out,
                          cudaStream_t s);
void launch_aos_to_planes(const double* in, long long count, double* re, double* im, cudaStream_t s);
void launch_step_once(const double* p, const double* v, double* out, std::size_t n,
                      cudaStream_t s);

// K3/K4/K5 fused per-trajectory sweep (k_sweep.cu)
std::size_t sweep_workspace(std::size_t d, int64_t batch);
// GRAPE chain: batched segment propagators, then the sequential chain (k_sweep.cu)
std::size_t grape_workspace(std::size_t d, int64_t segments);
void launch_grape(std::size_t d, const double* h0, const double* hc, const double* zero_h,
                  std::size_t n_ops, const double* ops, const double* amps, const double* zeros,
                  int64_t segments, int64_t steps_per_segment, double dt, double* x, void* work,
                  cudaStream_t s, cudaEvent_t ev_build_end);
// GRAPE chain for d = 9 in the real form (Hermitian rho0) (k_ptm.cu)
bool ptm_grape_supported(std::size_t d);
std::size_t ptm_grape_workspace(int64_t segments);
void launch_ptm_grape(const double* h0, const double* hc, const double* zero_h, std::size_t n_ops, const double* ops,
                      const double* amps, int64_t segments, int64_t steps_per_segment, double dt, double* rho,
                      void* work, cudaStream_t s, cudaEvent_t ev_build_end);
// GRAPE chain in the real transfer-matrix form (Hermitian rho0, n > 96) (k_grape_real.cu)
bool grape_real_supported(std::size_t d);
std::size_t grape_real_workspace(std::size_t d, int64_t segments);
void launch_grape_real(std::size_t d, const double* h0, const double* hc, const double* zero_h,
                       std::size_t n_ops, const double* ops, const double* amps, int64_t segments,
                       int64_t steps_per_segment, double dt, double* x_rho, int squaring_bound, void* work,
                       cudaStream_t s, cudaEvent_t ev_build_end);
void launch_sweep(std::size_t d, const double* h0, const double* hd, const double* hs,
                  std::size_t n_ops, const double* ops, const double* delta, const double* scale,
                  double dt, const double* rho0, int64_t batch, int64_t steps, double* pops,
                  double* ens_sum, void* work, cudaStream_t s);

// config 4 in the real (transfer-matrix) representation (k_ptm.cu)
bool ptm_sweep_supported(std::size_t d);
std::size_t ptm_sweep_workspace(int64_t batch);
void launch_ptm_sweep(std::size_t d, const double* h0, const double* hd, const double* hs,
                      std::size_t n_ops, const double* ops, const double* delta, const double* scale,
                      double dt, const double* rho0, int64_t batch, int64_t steps, double* pops,
                      double* ens_sum, void* work, cudaStream_t s);

// d <= 3 sweeps: warp-per-trajectory build, thread-per-trajectory stepping (k_ptm_small.cu)
bool ptm_small_supported(std::size_t d);
std::size_t ptm_small_workspace(std::size_t d, int64_t batch);
void launch_ptm_sweep_small(std::size_t d, const double* h0, const double* hd, const double* hs,
                            std::size_t n_ops, const double* ops, const double* delta, const double* scale,
                            double dt, const double* rho0, int64_t batch, int64_t steps, double* pops,
                            double* ens_sum, void* work, cudaStream_t s);

// end-to-end host-buffer evolve (host_pipeline.cu): chunked H2D / validation /
// steps / D2H pipeline; `step` runs one chunk on a compute stream
using ChunkWork = std::function<std::size_t(int64_t chunk)>;
using ChunkStep = std::function<void(const double* p_dev, double* x_dev, int64_t nb, void* work, cudaStream_t s)>;
void host_evolve(const double* p, std::size_t d, const double* rho0, int64_t batch, double* out, bool single,
                 const ChunkWork& work_bytes, const ChunkStep& step);

int sm_count();       // of the current device
int current_device();
// cudaFuncAttributeMaxDynamicSharedMemorySize, set once per (kernel, device)
void ensure_max_dyn_smem(const void* fn, int bytes);
// Wait for an event / a stream by polling (cudaEventQuery) instead of the
// runtime's blocking wait: a blocking cudaStreamSynchronize returned ~0.25-0.3 ms
// after the work completed on the GPU box (thread wake-up), which left the GPU
// idle mid-call (config-4 validation round trip) and padded every host-buffer call.
void sync_event_spin(cudaEvent_t e, const char* what);
void sync_stream_spin(cudaStream_t s, const char* what);

}  // namespace lbg
