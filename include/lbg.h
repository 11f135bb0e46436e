/*
 * lbg.h — C-ABI of the B200-native Lindblad propagation engine (liblbg.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv/paper_2603_18052 "lindbench", /root/reference/proj). Each entry point
 * names the reference interface it replaces (file:line, relative to proj/).
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *
 * Conventions:
 *  - complex128 matrices are row-major; "AoS" = interleaved (re, im) doubles
 *    exactly like lb::MatrixAoS (include/lb/complex_matrix.hpp:15-31); "SoA" =
 *    split re / im planes like lb::MatrixSoA (complex_matrix.hpp:35-45).
 *  - vec(rho) is row-major: rho[i][j] -> slot i*d + j (complex_matrix.hpp:78-81).
 *  - Functions suffixed _dev take DEVICE pointers, are stream-ordered and
 *    asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream)
 *    on the caller's current device. Everything else takes HOST pointers and is
 *    synchronous.
 *  - Status codes map 1:1 onto the reference's exception classes; no C++
 *    exception crosses the ABI. lbg_last_error() returns the calling thread's
 *    last message.
 */
#ifndef LBG_H
#define LBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBG_OK 0
#define LBG_EINVAL 1   /* std::invalid_argument (propagate.cpp:14-28, lindblad.cpp:25-33, expm.cpp:110-112) */
#define LBG_ERUNTIME 2 /* std::runtime_error (expm.cpp:40-41,120-121; propagate.cpp:65) */
#define LBG_ECUDA 3    /* CUDA launch / runtime failure (no reference counterpart) */

/* kernel selection for the batched shared-P stepper (0 = automatic) */
#define LBG_ALGO_AUTO 0
#define LBG_ALGO_CHAIN 1   /* K2: one warp, one trajectory, latency-bound (config 0) */
#define LBG_ALGO_DFMA9 2   /* K1a: n == 9, P in the constant bank, DFMA (config 1) */
#define LBG_ALGO_SMEM 3    /* K1b: n <= 84, P resident in shared memory, DMMA (config 2) */
#define LBG_ALGO_TILED 4   /* K1c: any n, P streamed from L2, persistent DMMA tiles (config 3) */
#define LBG_ALGO_CTA 5     /* K2b: n <= 96, one CTA per trajectory, P in shared memory (few trajectories) */
#define LBG_ALGO_ROWSPLIT 6 /* K2c: any n, batch <= 4, P's rows spread over all SMs' shared memory */
#define LBG_ALGO_CLUSTER 7  /* K1b-C: n == 81, 2-CTA clusters share a split n-tile through DSMEM */
#define LBG_ALGO_KSPLIT 8   /* K1b-K: n == 81, small batches: 2-CTA clusters split K, partials through DSMEM */

const char* lbg_last_error(void);
const char* lbg_version(void);

/* ------------------------------------------------------------------------
 * Raw step kernels — exact signatures of the reference's hot-loop pointers.
 * Replace lb::StepSoAFn (include/lb/kernels.hpp:23-24) and lb::StepAoSFn
 * (kernels.hpp:22; cplx* == interleaved double[2]). out[i] = sum_j P[i,j] v[j].
 * Host pointers; each call uploads P and v, runs one step on the GPU and
 * downloads `out` (compat shim for parity, not for speed). void return like
 * the reference; a CUDA failure aborts the process with a message (fail loud).
 * ------------------------------------------------------------------------ */
void lbg_step_soa(const double* p_re, const double* p_im, const double* v_re,
                  const double* v_im, double* out_re, double* out_im, size_t n);
void lbg_step_aos(const double* p, const double* v, double* out, size_t n);

/* ------------------------------------------------------------------------
 * Model assembly and propagator (device).
 * lbg_build_lindbladian_dev: replaces lb::build_lindbladian (lindblad.hpp:34,
 *   lindblad.cpp:37-59): L = -i(H(x)I - I(x)H^T) + sum_k [L_k(x)conj(L_k)
 *   - 1/2 L_k^dag L_k (x) I - 1/2 I (x) (L_k^dag L_k)^T], one thread per element.
 *   h: d*d AoS, ops: n_ops*d*d AoS, out: d^2*d^2 AoS (all device).
 *   Hermiticity of H is checked on the host side (lbg_build_lindbladian).
 * lbg_expm_dev: replaces lb::expm (expm.hpp:31, expm.cpp:109-134):
 *   P = exp(a*dt) for an n x n AoS matrix, by scaling and squaring around a
 *   degree-16 Taylor polynomial in Paterson-Stockmeyer form (6 DMMA matmuls,
 *   no solve; truncation <= 2^-54 relative for ||a dt||_1 <= 0.79 after
 *   scaling). `work` must hold 6*n*n complex (device).
 * ------------------------------------------------------------------------ */
int lbg_build_lindbladian(size_t d, const double* h, size_t n_ops, const double* ops,
                          double* out);
int lbg_build_lindbladian_dev(size_t d, const double* h, size_t n_ops, const double* ops,
                              double* out, void* stream);
int lbg_expm(const double* a, size_t n, double dt, double* out);
int lbg_expm_dev(const double* a, size_t n, double dt, double* out, double* work,
                 void* stream);
size_t lbg_expm_workspace(size_t n); /* bytes */

/* ------------------------------------------------------------------------
 * Batched building blocks (assemble / expm many independent
 * models at once, as a per-parameter sweep over arbitrary models needs —
 * propagate.cpp:137-143 builds one model, L and P per point):
 * lbg_build_lindbladian_batched_dev: out[b] = L(h[b], ops[b]) for b < batch;
 *   h: batch x d x d, ops: batch x n_ops x d x d, out: batch x d^2 x d^2
 *   (complex AoS, device); each out[b] is bit-identical to
 *   lbg_build_lindbladian_dev on model b (lindblad.cpp:37-59 order).
 * lbg_expm_batched_dev: out[b] = exp(a[b] dt) for b < batch (n x n each,
 *   device). n <= 16: one CTA per matrix with its own scaling (each out[b]
 *   equals lbg_expm_dev(a[b])); larger n: batched DMMA GEMMs with the batch's
 *   largest squaring count (within ~1e-14 of the per-matrix result). A
 *   non-finite entry anywhere -> LBG_EINVAL (expm.cpp:110-112); more than 64
 *   squarings -> LBG_ERUNTIME. Synchronises the stream once (the norm).
 *   `work` (device): lbg_expm_batched_workspace(n, batch) bytes.
 * ------------------------------------------------------------------------ */
int lbg_build_lindbladian_batched_dev(size_t d, const double* h, size_t n_ops, const double* ops,
                                      int64_t batch, double* out, void* stream);
size_t lbg_expm_batched_workspace(size_t n, int64_t batch); /* bytes */
int lbg_expm_batched_dev(const double* a, size_t n, int64_t batch, double dt, double* out, void* work,
                         void* stream);

/* ------------------------------------------------------------------------
 * Batched shared-P propagation: replaces lb::evolve (propagate.hpp:33-34,
 * propagate.cpp:75-109) over `batch` independent trajectories.
 * P: n x n AoS (n = d^2). X: batch x n complex, trajectory b's vec(rho_b) at
 * X[b*n ...]; SoA planes (x_re, x_im) or one AoS array. Updated in place after
 * `steps` steps. `algo` = LBG_ALGO_*. `work` (device) must hold
 * lbg_evolve_workspace(n, batch, algo) bytes (may be NULL when that is 0).
 * ------------------------------------------------------------------------ */
size_t lbg_evolve_workspace(size_t n, int64_t batch, int algo);
int lbg_evolve_shared_p_soa_dev(const double* p, size_t n, double* x_re, double* x_im,
                                int64_t batch, int64_t steps, int algo, void* work,
                                void* stream);
int lbg_evolve_shared_p_aos_dev(const double* p, size_t n, double* x, int64_t batch,
                                int64_t steps, int algo, void* work, void* stream);
/* the all-SoA form of the reference's Variant::soa (lb::Propagator::soa +
 * VectorSoA states, propagate.cpp:85-92): P as split re / im planes too.
 * work: lbg_evolve_planes_workspace(n, batch, algo) bytes (P is interleaved
 * into it on the device). */
size_t lbg_evolve_planes_workspace(size_t n, int64_t batch, int algo);
int lbg_evolve_shared_p_planes_dev(const double* p_re, const double* p_im, size_t n, double* x_re,
                                   double* x_im, int64_t batch, int64_t steps, int algo, void* work,
                                   void* stream);
/* host-buffer variant (end-to-end: H2D, steps, D2H; synchronous). rho0/out are
 * batch x d x d AoS density matrices; rho0 is validated like propagate.cpp:79. */
int lbg_evolve_shared_p(const double* p, size_t d, const double* rho0, int64_t batch,
                        int64_t steps, double* out, int algo);

/* ------------------------------------------------------------------------
 * Density-matrix mode of the same shared-P propagation (opt-in; the complex
 * entry points above stay the reference-faithful default). lb::evolve only
 * accepts physical states (propagate.cpp:77-80); a Lindblad propagator maps
 * Hermitian matrices to Hermitian matrices, so on the real coordinates
 * x[i*d+j] = Re rho_ij (i <= j), -Im rho_ij (i > j) it is the real matrix
 * P_R = T P T^-1 (4x fewer flops per step). rho = H + i H' with H, H'
 * Hermitian, propagated as two real vector sets. mode: LBG_DENSITY_HERMITIAN
 * asserts H' = 0 (rho stored exactly Hermitian, as GG^dag/tr is) and propagates
 * H only; LBG_DENSITY_GENERAL always propagates both; LBG_DENSITY_AUTO detects
 * H' != 0 on the device and skips the H' set when it is zero (no host sync).
 * P must preserve Hermiticity (every Lindblad propagator does). Any d: up to
 * d*d = 84 on the real register / shared-memory kernels, beyond on the real
 * variant of the K1c tile engine (n^2 FMAs per step everywhere; AUTO reads the
 * device flag there, one 4-byte sync). P: n x n AoS (device), rho: batch x d x d AoS
 * (device, in place), work: lbg_density_workspace(d*d, batch) bytes.
 * ------------------------------------------------------------------------ */
#define LBG_DENSITY_HERMITIAN 0
#define LBG_DENSITY_GENERAL 1
#define LBG_DENSITY_AUTO 2
size_t lbg_density_workspace(size_t n, int64_t batch);
int lbg_evolve_density_dev(const double* p, size_t d, double* rho, int64_t batch, int64_t steps,
                           int mode, void* work, void* stream);
/* host-buffer variant (end-to-end, synchronous, LBG_DENSITY_AUTO): rho0 / out
 * are batch x d x d AoS; rho0 is validated like propagate.cpp:79. */
int lbg_evolve_density(const double* p, size_t d, const double* rho0, int64_t batch,
                       int64_t steps, double* out);

/* ------------------------------------------------------------------------
 * Per-trajectory propagators (config 4, "robustness atlas"): for trajectory b
 *   H_b = h0 + delta[b] * hd + scale[b] * hs,   L_k fixed,
 *   L_b = build_lindbladian(H_b, L_k),  P_b = exp(L_b dt),
 *   rho_b <- P_b^steps rho0      (on the GPU: assembly K5, expm K4, stepping K3; in the
 *                                  default REAL mode the build exploits the sparse
 *                                  generator (K4-S) and P_R (52 KB per trajectory)
 *                                  passes through HBM once between K4 and K3)
 * Outputs: pops[b*d + i] = Re rho_b[i][i]; ens_sum (d*d AoS) += sum_b rho_b.
 * Replaces, per trajectory, the make_model + build_lindbladian + expm + step
 * sequence of lb::grape_chain (propagate.cpp:130-160). Device pointers.
 * mode: LBG_SWEEP_REAL propagates the real coordinates of the (Hermitian)
 * density matrix with the real d^2 x d^2 representation L_R = T L T^-1 of the
 * same generator (P_R = T P T^-1; 4x fewer flops; d == 9; rho0 must be exactly
 * Hermitian — checked on the device with the other input checks, one 32-byte
 * D2H per call). LBG_SWEEP_COMPLEX uses the
 * complex d^2 x d^2 matrices exactly as the reference does. AUTO = REAL when
 * it applies, else COMPLEX.
 * ------------------------------------------------------------------------ */
#define LBG_SWEEP_AUTO 0
#define LBG_SWEEP_COMPLEX 1
#define LBG_SWEEP_REAL 2
size_t lbg_sweep_workspace(size_t d, int64_t batch);
int lbg_evolve_sweep_dev(size_t d, const double* h0, const double* hd, const double* hs,
                         size_t n_ops, const double* ops, const double* delta,
                         const double* scale, double dt, const double* rho0, int64_t batch,
                         int64_t steps, double* pops, double* ens_sum, int mode, void* work,
                         void* stream);

/* ------------------------------------------------------------------------
 * GRAPE piecewise-constant chain: replaces lb::grape_chain (propagate.hpp:54-58,
 * propagate.cpp:111-168). Segment j evolves the state steps_per_segment steps
 * with P_j = exp(dt L(h0 + amplitudes[j] hc, ops)). All P_j are built in one
 * batched GPU pass (timed as build_ms), then the chain runs on the step kernels
 * (chain_ms), like ChainTimings (propagate.hpp:37-43). Host buffers: h0, hc
 * (d x d AoS), ops (n_ops x d x d), amplitudes (segments), rho0 / out (d x d).
 * rho0 must pass check_state (1e-8); h0 + a hc must be Hermitian (1e-12).
 * ------------------------------------------------------------------------ */
int lbg_grape_chain(size_t d, const double* h0, const double* hc, const double* amplitudes,
                    int64_t segments, int64_t steps_per_segment, double dt, size_t n_ops,
                    const double* ops, const double* rho0, double* out, double* build_ms,
                    double* chain_ms);

/* ------------------------------------------------------------------------
 * Batched invariant check: replaces lb::check_state (validate.hpp:22,
 * validate.cpp:10-30) over a batch. x: batch x d x d AoS (device).
 * Writes the max over the batch of |Tr rho - 1| and max|rho_ij - conj rho_ji|,
 * and the min Re rho_ii, into out3[0..2] (device).
 * ------------------------------------------------------------------------ */
int lbg_check_state_batched_dev(const double* x, size_t d, int64_t batch, double* out3,
                                void* stream);

/* ------------------------------------------------------------------------
 * Invariant checks with host buffers (validate.hpp:20-31, validate.cpp:10-45).
 * lbg_check_state: lb::check_state over `batch` d x d AoS states on the GPU
 *   (K6); out3 = {max |Tr rho - 1|, max |rho_ij - conj rho_ji|, min Re rho_ii}.
 * lbg_check_generator: lb::check_generator (validate.cpp:32-45): the states
 *   rho_t = lb::random_density(lb::make_rng(42), dim), t < trials, drawn in
 *   sequence as the reference does; *passed = 1 iff |Tr unvec(L vec(rho_t))|
 *   <= tol for all t (trace sums on the GPU); *worst (optional) = the largest
 *   |Tr|. L: rows x cols AoS; rows or cols != dim^2 -> LBG_EINVAL.
 * lbg_random_density_batch: lb::random_density drawn `count` times from
 *   lb::make_rng(seed) (random.hpp:12-37), count x d x d AoS.
 * lbg_validate_last_error(): message of the last failed call of this group.
 * ------------------------------------------------------------------------ */
const char* lbg_validate_last_error(void);
int lbg_check_state(const double* rho, size_t d, int64_t batch, double* out3);
int lbg_check_generator(size_t dim, const double* l, size_t rows, size_t cols, size_t trials, double tol,
                        int* passed, double* worst);
int lbg_random_density_batch(uint64_t seed, size_t d, int64_t count, double* out);

/* ------------------------------------------------------------------------
 * Ensemble reduction across ranks (config 4): in-place sum of `count` doubles
 * over the communicator `comm` (an ncclComm_t). The only collective of the
 * engine. Returns LBG_ECUDA if NCCL is unavailable.
 * ------------------------------------------------------------------------ */
int lbg_allreduce_sum_dev(double* buf, size_t count, void* comm, void* stream);
/* Ensemble mean of config 4 across ranks: buf (count doubles, each rank's
 * partial sum over its trajectories) is summed over `comm` (NULL = one rank, no
 * collective) and divided by the global trajectory count, in place. */
int lbg_ensemble_mean_dev(double* buf, size_t count, int64_t global_batch, void* comm, void* stream);
/* NCCL communicator plumbing (libnccl.so.2 is dlopen'ed on first use).
 * Rank 0 calls lbg_nccl_unique_id (128 bytes), the caller broadcasts the bytes
 * out of band (e.g. torch.distributed), then every rank calls
 * lbg_nccl_comm_init on its own device. */
int lbg_nccl_unique_id(void* id128);
int lbg_nccl_comm_init(void** comm, int nranks, const void* id128, int rank);
int lbg_nccl_comm_destroy(void* comm);

/* ------------------------------------------------------------------------
 * Host-side inputs (BASELINE.json configs). The
 * reference has no multi-transmon models, Ginibre states or sweeps; these are
 * built with the reference's primitives' arithmetic (kron, i-k-j matmul,
 * lindblad.cpp:76-80 lowering operator). cfg in 0..4.
 * ------------------------------------------------------------------------ */
int lbg_config_dims(int cfg, size_t* d, size_t* n_ops);
int lbg_config_model(int cfg, double delta, double s, double* h, double* ops);
/* config 4: H(delta, s) = h0 + delta*hd + s*hs (each 9x9 AoS) */
int lbg_config_sweep_terms(double* h0, double* hd, double* hs);
/* counter-based uniform in (0,1) keyed on (seed, cfg, trajectory, k) */
double lbg_uniform(uint64_t seed, uint32_t cfg, uint64_t traj, uint64_t k);
/* Ginibre rho0 (G with N(0,1) re/im by explicit Box-Muller, rho = GG^dag/tr)
 * for global trajectories [first, first+count): out is count x d x d AoS */
int lbg_ginibre_batch(uint64_t seed, uint32_t cfg, uint64_t first, int64_t count, size_t d,
                      double* out, int threads);
int lbg_sweep_params_batch(uint64_t seed, uint64_t first, int64_t count, double* delta,
                           double* scale);

/* ------------------------------------------------------------------------
 * Text formats of the reference (host only):
 *  lbg_write_matrix / lbg_read_matrix: the 17-significant-digit interchange
 *    format of lb::write_matrix / lb::read_matrix (complex_matrix.cpp:166-188);
 *    pass buf = NULL / out = NULL to query the size / shape first.
 *  lbg_read_model: lb::read_model (model_io.cpp:37-109): dim / hamiltonian /
 *    collapse keys or "preset = transmon" (lindblad.cpp:82-100). Call with
 *    h = ops = NULL to get d and n_ops, then with buffers (h: d*d, ops:
 *    cap_ops*d*d complex AoS).
 * Malformed text -> LBG_ERUNTIME, invalid model -> LBG_EINVAL;
 * lbg_io_last_error() has the message.
 * ------------------------------------------------------------------------ */
const char* lbg_io_last_error(void);
int lbg_write_matrix(const double* a, size_t rows, size_t cols, char* buf, size_t cap, size_t* len);
int lbg_read_matrix(const char* text, size_t* rows, size_t* cols, double* out, size_t cap_elems);
int lbg_read_model(const char* text, size_t* d, size_t* n_ops, double* h, double* ops, size_t cap_ops);

/* ------------------------------------------------------------------------
 * Kernel benchmark harness: replaces lb::run_bench / lb::write_csv /
 * lb::write_json (bench.hpp:14-37, bench.cpp:70-158, 202-248) for the GPU.
 * A bench is a chain of `warmup` untimed + `reps` timed steps of one random
 * P (uniform [-1,1] re/im from std::mt19937_64(seed), scaled by 1/d^2) on one
 * random vector, exactly the reference's inputs (bench.cpp:81-86,
 * random.hpp:12-22); `batch` (GPU extension, >= 1) runs that many copies of
 * the chain at once. checksum = sum of trajectory 0's final vector.
 * gflops = 8 d^4 / ns_per_step, gbs = 16 (d^4 + 2 d^2) / ns_per_step
 * (roofline.cpp:62-74). variant: LBG_VARIANT_AOS / SOA (kernels.hpp:15);
 * LBG_VARIANT_SIMD is the reference's AVX2 path and fails with LBG_ERUNTIME
 * like an unavailable variant (bench.cpp:77-78).
 * lbg_run_bench: timed with CUDA events around the `reps` steps. Errors also
 * set out->failed and out->error (for the writers' "# failed" rows).
 * lbg_write_bench_csv / _json: the reference's report formats (same columns
 * / keys, same number formatting) plus the GPU columns batch, algo,
 * traj_steps_per_s; buf = NULL queries *len.
 * ------------------------------------------------------------------------ */
#define LBG_VARIANT_AOS 0
#define LBG_VARIANT_SOA 1
#define LBG_VARIANT_SIMD 2
typedef struct {
  size_t dim;
  int variant;
  int64_t reps, warmup;
  uint64_t seed;
  int64_t batch;
} lbg_bench_config;
typedef struct {
  double ns_per_step, gflops, gbs, checksum_re, checksum_im, traj_steps_per_s;
  int algo, failed;
  char error[224];
} lbg_bench_result;
const char* lbg_bench_last_error(void); /* message of the last failed inputs / writer call */
int lbg_bench_inputs(size_t dim, uint64_t seed, double* p, double* v0);
int lbg_run_bench(const lbg_bench_config* cfg, lbg_bench_result* out);
int lbg_write_bench_csv(const lbg_bench_config* cfgs, const lbg_bench_result* res, size_t count,
                        const char* machine, char* buf, size_t cap, size_t* len);
int lbg_write_bench_json(const lbg_bench_config* cfgs, const lbg_bench_result* res, size_t count,
                         const char* machine, char* buf, size_t cap, size_t* len);

/* ------------------------------------------------------------------------
 * Roofline model on the GPU: replaces lb::characterize / place / classify /
 * ridge_point, lb::MachineProfile and its text format (roofline.hpp:11-80,
 * roofline.cpp:44-182). The B200 ladder fills the reference's 4-level shape:
 *   level 0 "L1"   shared memory per SM (capacity: bytes per SM),
 *   level 1 "L2"   L2 cache,
 *   level 2 "L3"   HBM,
 *   level 3 "DRAM" host memory over PCIe (pinned H2D),
 * peak_gflops = FP64 (DMMA) peak. lbg_measure_machine_profile measures every
 * number on the current device; lbg_write/read_machine_profile use the
 * reference's "key = value" file (peak_gflops, bw_l1..bw_dram GB/s,
 * cap_l1..cap_l3 bytes), so lb::read_profile loads a B200 profile and the
 * reference's own place/classify run against it. Characterize / place /
 * classify follow the reference exactly (8 d^4 flops, 16 (d^4 + 2 d^2) bytes,
 * smallest level whose capacity holds the working set, memory bound iff
 * ai < peak / bw). Invalid profiles -> LBG_EINVAL, malformed text ->
 * LBG_ERUNTIME; lbg_roofline_last_error() has the message.
 * ------------------------------------------------------------------------ */
typedef struct {
  char name[64];
  double peak_gflops;
  double bandwidth_gbs[4];
  uint64_t capacity_bytes[3];
} lbg_machine_profile;
typedef struct {
  size_t dim;
  uint64_t flops, bytes;
  double ai;
  uint64_t working_set_bytes;
  int placement; /* 0..3 = L1, L2, L3, DRAM; -1 = unset */
} lbg_kernel_character;
#define LBG_MEMORY_BOUND 0
#define LBG_COMPUTE_BOUND 1
const char* lbg_roofline_last_error(void);
int lbg_measure_machine_profile(lbg_machine_profile* out);
int lbg_validate_profile(const lbg_machine_profile* m);
int lbg_characterize(size_t d, lbg_kernel_character* out);
int lbg_place(lbg_kernel_character* k, const lbg_machine_profile* m);
int lbg_ridge_point(const lbg_machine_profile* m, int level, double* out);
int lbg_classify(const lbg_kernel_character* k, const lbg_machine_profile* m, int* bound,
                 double* attainable_gflops);
int lbg_write_machine_profile(const lbg_machine_profile* m, char* buf, size_t cap, size_t* len);
int lbg_read_machine_profile(const char* text, const char* name, lbg_machine_profile* out);

/* FP64 roofline denominators measured live on the current device (TF/s):
 * register-only DMMA (m8n8k4 f64) and DFMA loops over every SM. */
int lbg_fp64_peak(double* dmma_tflops, double* dfma_tflops);

/* Number of kernels this thread launched since the last reset (evidence for
 * bench.py's gpu_launches). */
int64_t lbg_launch_count(void);
void lbg_reset_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LBG_H */
