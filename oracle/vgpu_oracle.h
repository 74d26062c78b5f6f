/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by or called
 * from the product path (paper_1511_07658_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, as the checker.
 *
 * CPU restatements of the reference's arithmetic for the GVM hot path:
 *   vector add / scale   proj/src/payload_kernels.cpp:13-16, :24-27 (serial twins)
 *                        — PINNED: bit-exact vs the reference itself (oracle/_ref)
 *                          and its goldens (proj/tests/test_payload.cpp:26-79).
 *   NAS EP               no reference arithmetic (proj/src/bench/profiles.cpp:27,:31 are
 *                        timing-only); restated from NPB 3.x EP (ep.f) —
 *                        PINNED against the published NPB verification sums
 *                        (classes S, W, A; epsilon 1e-8) in tests/golden/.
 *   Black-Scholes        no reference arithmetic (profiles.cpp:39); CUDA-SDK
 *                        formulation in binary64 — UNPINNED by the reference
 *                        itself; pinned instead to a published worked example
 *                        (Hull Ex. 15.6) and the exact-CDF closed form
 *                        (tests/test_oracle.py). GPU checked at L1 rel <= 1e-6.
 *   NAS CG               no reference arithmetic (profiles.cpp:41); NPB 3.x cg.f
 *                        makea + conj_grad — PINNED against NPB's published
 *                        zeta (classes S, W, A; epsilon 1e-10).
 *   Electrostatics       no reference arithmetic (profiles.cpp:43); binary64
 *                        direct Coulomb sum — UNPINNED by the reference; pinned
 *                        to the single-charge closed form and superposition.
 *   SGEMM                no reference arithmetic (profiles.cpp:35); binary64
 *                        accumulation — UNPINNED by the reference itself;
 *                        pinned to numpy float64 matmul and exact integer
 *                        products. GPU checked at relative Frobenius <= 1e-5.
 */
#ifndef VGPU_ORACLE_H
#define VGPU_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/vgpu_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

void vo_vector_add(float* out, const float* a, const float* b, size_t n);
void vo_vector_scale(float* out, const float* in, float factor, size_t n);
void vo_vector_mul(float* out, const float* a, const float* b, size_t n);

/* One EP job with the documented fixed reduction order:
 * 256 lanes per batch, each lane sums its pairs sequentially, lanes combine
 * in a binary tree, batches accumulate sequentially in batch order. */
/* NAS EP job in the kernel's reduction order (accepted pairs compacted per
 * warp); vo_ep_job_lanes: the lane-sequential order of the
 * branch-free kernel instance (VGPU_EP_VARIANT=11) */
int vo_ep_job(const vgpu_ep_params* p, vgpu_ep_result* r);
int vo_ep_job_lanes(const vgpu_ep_params* p, vgpu_ep_result* r);
/* Fold job results in order (the GVM / rank-order host fold). */
/* vgpu_ep_log (ep_math.h, shared with the kernel) over an array: accuracy tests */
void vo_ep_log(const double* x, double* y, size_t n);
void vo_ep_fold(const vgpu_ep_result* parts, size_t n, vgpu_ep_result* out);

void vo_black_scholes(const float* S, const float* X, const float* T, size_t n,
                      double riskfree, double volatility, double* call, double* put);

void vo_sgemm(const float* A, const float* B, size_t n, double* C);

/* NAS CG: NPB makea into the nas-cg input layout (returns the bytes needed;
 * writes when out has room) and the timed CG iterations on such an input
 * (nonzero on a malformed input). */
uint64_t vo_cg_makea(uint32_t n, uint32_t nonzer, uint32_t niter, double shift, uint8_t* out,
                     uint64_t cap);
int vo_cg_run(const uint8_t* in, uint64_t in_bytes, vgpu_cg_result* res);

/* Electrostatics: binary64 lattice potential of an "electrostatics" input
 * (out: nx*ny*nz doubles); nonzero on a malformed input. */
int vo_es(const uint8_t* in, uint64_t in_bytes, double* out);

/* deterministic generators shared by tests and bench (xorshift64*) */
/* NAS MG (NPB 3.x mg.f): zran3's right-hand side as the nas-mg input
 * (returns the bytes needed; writes when cap suffices), and the timed part
 * (resid, nit x (mg3P, resid), norm2u3). u_top (optional): the finest u
 * with its ghost layer, (nx + 2)^3 doubles, for bit-exact grid checks. */
uint64_t vo_mg_make_input(uint32_t nx, uint32_t nit, uint32_t coeffs, uint8_t* out, uint64_t cap);
int vo_mg_run(const uint8_t* in, uint64_t bytes, vgpu_mg_result* res, double* u_top);

uint64_t vo_rng_next(uint64_t* state);
float vo_rng_uniform(uint64_t* state, float lo, float hi);

#ifdef __cplusplus
}
#endif

#endif
