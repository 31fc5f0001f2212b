/*
 * ietidp_shard.h — C ABI of the sharded (multi-GPU) solve phase (libietidp.so; SURVEY §8(e),
 * §8(f) row f4). Citations "P:<line>" are lines of /root/reference/PAPER.md.
 *
 * The subdomains are the units of parallelism of the IETI-DP method: each
 * rank (one process per GPU) owns a subset, factors and stores only those, and the ranks
 * exchange
 *   set-up:     the K diagonals on the multipliers' two sides (stiffness scaling),
 *               S_PP (n_primal^2) and ftilde (n_primal x nrhs)             -- P:134
 *               d_DP (n_lambda x nrhs)                                      -- P:136-139
 *   per PCG iteration: the coarse right-hand side g = sum_k C_k^T G_k^T B^T p
 *               (n_primal x nrhs), the product q = F_DP p and the preconditioned residual
 *               z = M_D^-1 r (n_lambda x nrhs each)                         -- P:128
 *   recovery:   g for the coarse solution (n_primal x nrhs)                 -- P:129
 * each as ONE sum over the ranks of a device buffer (an all-reduce). The multiplier-space
 * vectors (lambda, r, p, q, z) and S_PP^-1 are replicated, so the CG scalars and the
 * stopping decisions are computed redundantly and identically on every rank: no scalar
 * exchange is needed.
 *
 * A sharded handle is an ordinary handle (ietidp.h) created with the rank's LOCAL subdomain
 * count and the GLOBAL n_lambda, n_primal, nrhs; the rank's subdomains are set with local
 * ids 0 .. n_local-1 and global multiplier / primal ids. Multiplier rows with one side (or
 * none) on this rank are legal in sharded mode. ietidp_factor / ietidp_solve / ietidp_get_u /
 * ietidp_apply_F / ietidp_apply_precond then work as documented in ietidp.h, collectively:
 * every rank must make the same calls in the same order. Sharded mode runs the explicit loop
 * with the residual stopping criterion, launch by launch (no persistent kernel: its grid
 * barrier cannot span GPUs).
 */
#ifndef IETIDP_SHARD_H
#define IETIDP_SHARD_H

#include <stdint.h>

#include "ietidp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* In-place sum over all ranks of the device buffer d_buf[0..n) (FP64). Called by the library
 * with all producing work already enqueued on `stream` (a cudaStream_t); the implementation
 * must order itself after that work and before work enqueued on `stream` later (an NCCL
 * all-reduce on `stream` does; a host-staged implementation synchronises the stream). The
 * result must be bitwise identical on every rank. Returns 0 on success. */
typedef int (*ietidp_allreduce_fn)(void* ctx, double* d_buf, int64_t n, void* stream);

/* Switch the handle to sharded mode; before ietidp_analyze. rank in [0, nranks).
 * Errors: E_ARG (null fn, rank out of range, triangular loop or preconditioned stopping
 * selected), E_STATE (after analysis). */
ietidp_status ietidp_shard_enable(ietidp_t h, int rank, int nranks, ietidp_allreduce_fn fn, void* ctx);

/* The same with NCCL as the transport, called from the library without leaving native code:
 * nccl_comm is the rank's ncclComm_t and nccl_allreduce the address of ncclAllReduce in the
 * NCCL library the caller has loaded (the library itself does not link NCCL). Every sum is
 * one ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, comm, stream) on the library's stream:
 * over NVLink 5 / NVSwitch, in-switch reduction (NVLS) where NCCL enables it.
 * Errors as ietidp_shard_enable. */
ietidp_status ietidp_shard_enable_nccl(ietidp_t h, int rank, int nranks, void* nccl_comm, void* nccl_allreduce);

/* Contiguous partition of n_sub subdomains over nranks ranks balanced by weight[k] > 0
 * (e.g. factor flops + loop bytes): owner[k] in [0, nranks), non-decreasing in
 * k; every rank gets at least one subdomain when n_sub >= nranks. Host only (no device).
 * Greedy prefix cuts at the multiples of the mean weight. Errors: E_ARG. */
ietidp_status ietidp_shard_partition(int n_sub, const double* weight, int nranks, int32_t* owner);

#ifdef __cplusplus
}
#endif
#endif /* IETIDP_SHARD_H */
