/*
 * cstress_b200.h -- C-ABI of the B200-native MSET2 path.
 *
 * Drop-in boundary for the reference's train/estimate plugin
 * (/root/reference/proj/include/containerstress/estimator.hpp:18-29) and the
 * per-op backend entry points its tests call directly
 * (backends.hpp:46-65).  Plain pointers and sizes only; every matrix is
 * column-major FP64 on the host, exactly the reference's Eigen layout
 * (types.hpp:7-15).  Signal matrices are observations x signals
 * (signals.hpp:45-51), memory matrices signals x memory vectors
 * (mset.hpp:21-27).
 *
 * Errors: every entry point returns a cs_status that maps 1:1 onto the
 * reference exception classes (errors.hpp:9-74); cs_last_error() returns the
 * thread-local message, reproducing the reference texts (e.g.
 * "select_memory_vectors: m=3 violates m >= 2n with n=2", mset.cpp:77-79).
 * CUDA / out-of-memory failures map to CS_ERROR (the `Error` base class).
 *
 * Threading: one cs_ctx (device + stream + workspace) per host thread.
 * Every host-buffer call is synchronous on return (run_cell brackets wall
 * time around train/estimate, sweep.cpp:212-219).  A cs_model is immutable
 * after training and may be used from several contexts on its device
 * (mset.hpp:45).
 */
#ifndef CSTRESS_B200_H
#define CSTRESS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CS_OK = 0,
  CS_ERROR = 1,                 /* cstress::Error (incl. CUDA / OOM)          */
  CS_CONSTRAINT_VIOLATED = 2,   /* ConstraintViolated   errors.hpp:28-31       */
  CS_INSUFFICIENT_TRAINING = 3, /* InsufficientTraining errors.hpp:32-35       */
  CS_DEGENERATE_MODEL = 4,      /* DegenerateModel      errors.hpp:36-39       */
  CS_EIG_FAILURE = 5,           /* EigFailure           errors.hpp:40-43       */
  CS_SHAPE_ERROR = 6,           /* ShapeError           errors.hpp:46-49       */
  CS_CONFIG_ERROR = 7,          /* ConfigError          errors.hpp:66-69       */
  CS_IO_ERROR = 8,              /* IoError              errors.hpp:70-73       */
  CS_MOMENT_INFEASIBLE = 9,     /* MomentInfeasible     errors.hpp:15-18       */
  CS_BAD_CORRELATION = 10,      /* BadCorrelation       errors.hpp:19-22       */
  CS_TOO_FEW_SAMPLES = 11,      /* TooFewSamples        errors.hpp:23-26       */
  CS_EMPTY_GRID = 12            /* EmptyGrid            errors.hpp:52-55       */
} cs_status;

/* KernelKind (kernels.hpp:12) */
enum { CS_KERNEL_INVERSE_DISTANCE = 0, CS_KERNEL_GAUSSIAN = 1 };

/* Surveillance arithmetic.
 *  CS_PRECISION_FP64: reference association (W = G+ S, est = D W,
 *    mset.cpp:189-192) in FP64 with the reference's summation order and no
 *    FMA contraction -- bit-identical to the CPU reference given the same model.
 *  CS_PRECISION_FP32: reassociated est = P S with P = D_norm G+ formed once at
 *    train time in FP64, distance and weight GEMMs on tcgen05
 *    tensor cores as 3xFP16 split products (FP32-accurate), kernel map fused
 *    in the epilogue.  Tolerance 1e-3 relative to max|estimate| (north_star). */
enum { CS_PRECISION_FP64 = 0, CS_PRECISION_FP32 = 1 };

/* Element types for device-resident I/O. */
enum { CS_DTYPE_F64 = 0, CS_DTYPE_F32 = 1 };

typedef struct cs_ctx cs_ctx;
typedef struct cs_model cs_model;

const char* cs_last_error(void);
const char* cs_version(void);

/* ----------------------------------------------------------- contexts */
cs_status cs_ctx_create(int device, cs_ctx** out);
cs_status cs_ctx_destroy(cs_ctx* ctx);
/* Run on an external cudaStream_t (e.g. torch's current stream); NULL is
 * the legacy default stream.  cs_ctx_reset_stream restores the context's
 * own non-blocking stream. */
cs_status cs_ctx_set_stream(cs_ctx* ctx, void* cuda_stream);
cs_status cs_ctx_reset_stream(cs_ctx* ctx);
cs_status cs_ctx_synchronize(cs_ctx* ctx);
/* Device name / SM count / arithmetic description (BackendCapabilities,
 * backends.hpp:35-41). */
cs_status cs_ctx_describe(cs_ctx* ctx, char* buf, size_t buflen);

/* ------------------------------------------------------ per-op entry points
 * Host buffers, synchronous.  Replace sim_matrix / matmul / batched_solve
 * (backends.hpp:46-65, backends.cpp:206-213, :276-293) and symmetric_eig
 * (mset.hpp:34-38).  bandwidth <= 0 means "unset" -> sqrt(n)
 * (KernelConfig::resolved, kernels.hpp:30-34).  FP64 with the reference's
 * accumulation order: bit-identical to sim_matrix_reference for the
 * inverse-distance kernel and to matmul_reference for every input. */
cs_status cs_sim_matrix(cs_ctx* ctx, const double* A, const double* B,
                        int64_t n, int64_t p, int64_t q, int kernel_kind,
                        double bandwidth, double* out /* p x q */);
cs_status cs_matmul(cs_ctx* ctx, const double* A /* p x k */,
                    const double* B /* k x q */, int64_t p, int64_t k,
                    int64_t q, double* out /* p x q */);
cs_status cs_batched_solve(cs_ctx* ctx, const double* G_pinv /* m x m */,
                           const double* S /* m x q */, int64_t m, int64_t q,
                           double* out /* m x q */);
cs_status cs_symmetric_eig(cs_ctx* ctx, const double* G, int64_t m,
                           double* eigenvalues /* m, ascending */,
                           double* eigenvectors /* m x m */);

/* Eigenvalues only (ascending) of a symmetric m x m matrix -- the
 * eigen_spectrum part of symmetric_eig (mset.cpp:57-70), same precondition
 * (ShapeError when not symmetric to 1e-9).  For m <= 2048 the library's own
 * shared-memory tridiagonalisation + Sturm multisection (exact to 1e-12 of
 * max|lambda|, faster than syevd at every size there; CSB_EIG_OWN=0 forces
 * syevd), cuSOLVER syevd above. */
cs_status cs_symmetric_eigvals(cs_ctx* ctx, const double* G, int64_t m, double* w);

/* select_memory_vectors (mset.cpp:72-137): bit-exact indices. */
cs_status cs_select_memory_vectors(cs_ctx* ctx, const double* training,
                                   int64_t N, int64_t n, int64_t m,
                                   int64_t* source_indices /* m */,
                                   double* D /* n x m, may be NULL */);

/* ----------------------------------------------------- train / estimate
 * cs_mset_train replaces cstress::train (mset.cpp:139-172) /
 * MsetAlgorithm::train (estimator.cpp:27-33). */
cs_status cs_mset_train(cs_ctx* ctx, const double* training /* N x n */,
                        int64_t N, int64_t n, int64_t m, int kernel_kind,
                        double bandwidth, int precision, cs_model** out);
/* Device-resident training input (col-major FP64 N x n on ctx's device). */
cs_status cs_mset_train_device(cs_ctx* ctx, const double* d_training,
                               int64_t N, int64_t n, int64_t m,
                               int kernel_kind, double bandwidth,
                               int precision, cs_model** out);

/* cs_mset_estimate replaces cstress::estimate (mset.cpp:174-199) /
 * MsetAlgorithm::estimate (estimator.cpp:35-40): host FP64 observations in,
 * host FP64 estimates and residuals out (either may be NULL).  H2D, compute
 * and D2H are pipelined over observation chunks on two streams. */
cs_status cs_mset_estimate(cs_ctx* ctx, const cs_model* model,
                           const double* observations /* N x n */, int64_t N,
                           int64_t n, double* estimates /* N x n */,
                           double* residuals /* N x n */);
/* Device-resident variant: observations / estimates / residuals are
 * column-major N x n device arrays of `io_dtype` with leading dimension ld
 * (>= N).  Asynchronous on the context stream. */
cs_status cs_mset_estimate_device(cs_ctx* ctx, const cs_model* model,
                                  const void* d_observations, int io_dtype,
                                  int64_t N, int64_t n, int64_t ld,
                                  void* d_estimates, void* d_residuals);

/* Model introspection / export (TrainedModel fields, mset.hpp:46-57). */
cs_status cs_model_info(const cs_model* model, int64_t* n_signals,
                        int64_t* n_memory, int64_t* rank, int* kernel_kind,
                        double* bandwidth, int* precision);
cs_status cs_model_export(const cs_model* model, int64_t* source_indices,
                          double* D, double* gram_pinv, double* eigen_spectrum,
                          double* signal_scale);
/* Host TrainedModel -> device model (the load_model path, mset.cpp:269-310). */
cs_status cs_model_import(cs_ctx* ctx, int64_t n, int64_t m, int kernel_kind,
                          double bandwidth, int64_t rank,
                          const int64_t* source_indices, const double* D,
                          const double* gram_pinv, const double* eigen_spectrum,
                          const double* signal_scale, int precision,
                          cs_model** out);
cs_status cs_model_destroy(cs_model* model);

/* Model wire format (multi-GPU C5'): the whole device model --
 * header, source indices, spectrum, D, D_norm, scale, G+, and the packed
 * FP32 tensor-core operand tiles -- as ONE contiguous device buffer, so a
 * trained model moves between GPUs with a single collective (NCCL
 * broadcast over NVLink) and no host round trip.  No reference counterpart:
 * the reference trains and estimates in one process on one host
 * (mset.cpp:139-199); this is the broadcast step of "train once, shard the
 * observations".  Unpacking copies into a new model on ctx's device whose
 * estimates are bitwise those of the packed model.  Errors: CS_CONFIG_ERROR
 * for a short buffer, CS_IO_ERROR for a buffer that is not a model wire. */
cs_status cs_model_wire_size(const cs_model* model, int64_t* bytes);
cs_status cs_model_pack_device(cs_ctx* ctx, const cs_model* model,
                               void* d_wire, int64_t bytes);
cs_status cs_model_unpack_device(cs_ctx* ctx, const void* d_wire,
                                 int64_t bytes, cs_model** out);

/* CSM1 model files (save_model / load_model, mset.cpp:225-310; declared at
 * mset.hpp:83-86): byte-compatible with the reference writer, including the
 * "<path>.json" sidecar.  Errors: CS_IO_ERROR with the reference texts
 * ("load_model: bad magic in <path>", "... truncated file ...", ...). */
cs_status cs_model_save(const cs_model* model, const char* path);
cs_status cs_model_load(cs_ctx* ctx, const char* path, int precision,
                        cs_model** out);

/* ------------------------------------------------------------------ SPRT
 * Wald sequential probability ratio test on residual streams (north_star
 * "SPRT alarm flags").  NOT in the reference, so the
 * definition is this project's, checked bit-for-bit against
 * oracle/cstress_oracle.c:or_sprt (parity against the reference: unpinned).
 * Per signal s: positive test lambda += c[s]*(r - h[s]), negative test
 * lambda += c[s]*((-r) - h[s]) (FP64, that operation order, no FMA);
 * lambda >= B -> alarm (flags bit 0 / bit 1) and lambda = 0; lambda <= A ->
 * lambda = 0.  Typical: M = k sigma, c = M / sigma^2, h = M / 2,
 * A = ln(beta / (1 - alpha)), B = ln((1 - beta) / alpha).
 * state: 2 doubles per signal (positive, negative), carried across calls.
 * flags: N x n column-major uint8; counts: 2 per signal (may be NULL). */
cs_status cs_sprt(cs_ctx* ctx, const double* residuals /* N x n host */,
                  int64_t N, int64_t n, const double* c, const double* h,
                  double A, double B, double* state, uint8_t* flags,
                  int64_t* counts);
/* residuals on the device (FP64 or FP32, leading dimension ld); flags on
 * the device (leading dimension N); c, h, state, counts on the host. */
cs_status cs_sprt_device(cs_ctx* ctx, const void* d_residuals, int dtype,
                         int64_t N, int64_t n, int64_t ld, const double* c,
                         const double* h, double A, double B, double* state,
                         uint8_t* d_flags, int64_t* counts);

/* ------------------------------------------------------------ data feed
 * synthesize (signals.cpp:205-254) for SignalSpec::uniform (signals.cpp:51-65),
 * host FP64 output N x n.  Seeds per rng.hpp:26-33. */
cs_status cs_synthesize_uniform(int64_t n, int64_t N, double phi, double rho,
                                double variance, double skewness,
                                double kurtosis, uint64_t seed, double* out);
/* Same recipe on the device (d_out: column-major N x n FP64 on ctx's device):
 * counter-based Box-Muller draws, chunked AR(1) scan, O(N n) mixing with the
 * closed-form compound-symmetric Cholesky factor.  Tolerance parity with the
 * host feed (libm / summation order differ in the last bits).  Synchronous. */
cs_status cs_synthesize_uniform_device(cs_ctx* ctx, int64_t n, int64_t N, double phi,
                                       double rho, double variance, double skewness,
                                       double kurtosis, uint64_t seed, double* d_out);
/* Same feed, FP32 result: d_work (N x n FP64 scratch) holds the FP64 stream
 * and the final variance-scale pass writes (float)(x * scale) into d_out32
 * -- bit-identical to converting cs_synthesize_uniform_device's output,
 * without the extra FP64 write and conversion pass (device-resident FP32
 * surveillance blocks for the sweep).  Synchronous. */
cs_status cs_synthesize_uniform_device_f32(cs_ctx* ctx, int64_t n, int64_t N, double phi,
                                           double rho, double variance, double skewness,
                                           double kurtosis, uint64_t seed, double* d_work,
                                           float* d_out32);
uint64_t cs_derive_seed(uint64_t parent, const uint64_t* coords, int ncoords);
/* sweep.cpp:119-126 */
uint64_t cs_cell_data_seed(uint64_t master_seed, int64_t n_signals,
                           int64_t n_observations, int64_t n_memory,
                           int replicate);

#ifdef __cplusplus
}
#endif
#endif /* CSTRESS_B200_H */
