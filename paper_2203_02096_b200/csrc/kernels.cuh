// kernels.cuh — host-side launchers of the sm_100a kernels (implemented in kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dock_internal.h"

namespace dk {

// Scratch layout of one lane group (bytes, 16-aligned offsets).
struct ScratchLayout {
    int off_r, off_W, off_tp, off_ts, off_genes, off_grad, off_extra, bytes;
};

// Local-search launch arguments.  use_state = 1: engine mode (per-run state decides the
// generation, buffers and the LS pick); 0: parity-hook mode on a plain [n][G] array.
struct LsArgs {
    int use_state;
    int n_per_run;          // LS individuals per run
    int iters;
    float *genes;           // hook mode: [n][G]
    float *E;               // hook mode: [n]
    int *evals;             // hook mode: [n] evaluation counts (engine: PopDev.ls_evals)
    const int *rng_slot;    // hook mode: [n] population index used as SW RNG slot
    int gen, run;           // hook mode: generation and global run index
    int wave_total;         // LS individuals in flight on the device for the speculation-depth rule
                            // (per-run launches of concurrent branches: all runs'); 0 = this launch's
    // Solis-Wets "fed" parity mode (hook mode only; SURVEY §8(c) parity protocol): the energy
    // of candidate c (0 = x+b+d, 1 = x-b-d) of iteration it of individual i is
    // sw_fed[(i iters + it) 2 + c] instead of the evaluation's, so the D9 state machine is
    // compared with the oracle's on identical energies.  sw_trace / sw_trace_rho [n][iters]:
    // outcome (0, 1, 2) and rho of every executed iteration.  All null in production.
    const float *sw_fed;
    int *sw_trace;
    float *sw_trace_rho;
    // ADADELTA parity mode (hook mode only): ad_fed [n][iters][1+G] replaces iteration it's
    // (energy, gradient) of individual i; ad_trace_x / ad_trace_g [n][iters][G] and
    // ad_trace_E [n][iters] receive the point evaluated at every iteration, its gradient and
    // its energy (the kernel's own, or the fed ones).  All null in production.
    const float *ad_fed;
    float *ad_trace_x, *ad_trace_E, *ad_trace_g;
};

struct GroupCfg {
    int W;      // lanes per individual (16 or 32)
    int MAXC;   // atom chunks per lane (1, 2, 4, 8)
};
// The kernels are compiled once per scoring function (score.cuh): dk::d5 (D5) and
// dk::ad4 (NEXT-2, D5-AD4).  Each namespace declares the same launchers; the dk:: wrappers
// below pick one by LigDev::sf, so the engine's call sites do not change.
#define DK_LAUNCHER_DECLS                                                                                    \
    GroupCfg pick_group(int N);                                                                              \
    ScratchLayout scratch_layout(const LigDev &L, bool grad, int extra_bytes);                               \
    cudaError_t setup_kernel_attributes();                                                                   \
    cudaError_t launch_eval(const LigDev &L, const GridDev &g, int n, const float *genes, float *E,          \
                            float *grad, float *xyz, const int *dfs2orig, cudaStream_t s, int parts);        \
    cudaError_t launch_init(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,       \
                            cudaStream_t s);                                                                 \
    cudaError_t launch_ga(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,         \
                          int *dbg, cudaStream_t s);                                                         \
    cudaError_t launch_ls(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,         \
                          const LsArgs &a, int n_total, cudaStream_t s);                                     \
    int run_sw_eligible(const LigDev &L, const SearchDev &sp);                                               \
    int adadelta_resident_groups(const LigDev &L);                                                           \
    cudaError_t launch_run_sw(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,     \
                              unsigned long long *prof, cudaStream_t s);                                     \
    cudaError_t launch_bench_part(const LigDev &L, const GridDev &g, int part, int n, int iters,             \
                                  const float *genes, float *E, cudaStream_t s);                             \
    cudaError_t launch_gen_end(const SearchDev &sp, const PopDev &pop, cudaStream_t s);                      \
    cudaError_t launch_best(const LigDev &L, const SearchDev &sp, const PopDev &pop, float *bestE,           \
                            float *bestG, long long *evals, int *gens, cudaStream_t s);                      \
    cudaError_t launch_philox(int n, const uint32_t *ctr, const uint32_t *key, uint32_t *out, cudaStream_t s); \
    cudaError_t launch_l2_gather(const float4 *buf, uint32_t n, int blocks, int iters, float *out, cudaStream_t s); \
    cudaError_t launch_stream_words(uint32_t k0, uint32_t k1, uint32_t purpose, uint32_t slot, uint32_t gen, \
                                    uint32_t run, uint32_t m0, int n, uint32_t *out, cudaStream_t s);
namespace d5 { DK_LAUNCHER_DECLS }
namespace ad4 { DK_LAUNCHER_DECLS }
#undef DK_LAUNCHER_DECLS

enum { kScoreD5 = 0, kScoreAD4 = 1 };
#ifndef DK_KERNELS_TU   // the dispatching wrappers are for the engine, not for kernels.cu (ADL)
// energy parts for launch_eval (score.cuh kInter / kIntra / kAll)
enum { kPartsInter = 1, kPartsIntra = 2, kPartsAll = 3 };

inline GroupCfg pick_group(int N) { return d5::pick_group(N); }
inline ScratchLayout scratch_layout(const LigDev &L, bool grad, int extra_bytes) {
    return d5::scratch_layout(L, grad, extra_bytes);
}
inline cudaError_t setup_kernel_attributes() {
    const cudaError_t e = d5::setup_kernel_attributes();
    return e != cudaSuccess ? e : ad4::setup_kernel_attributes();
}
inline cudaError_t launch_eval(const LigDev &L, const GridDev &g, int n, const float *genes, float *E,
                               float *grad, float *xyz, const int *dfs2orig, cudaStream_t s,
                               int parts = kPartsAll) {
    return L.sf == kScoreAD4 ? ad4::launch_eval(L, g, n, genes, E, grad, xyz, dfs2orig, s, parts)
                             : d5::launch_eval(L, g, n, genes, E, grad, xyz, dfs2orig, s, parts);
}
inline cudaError_t launch_init(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                               cudaStream_t s) {
    return L.sf == kScoreAD4 ? ad4::launch_init(L, g, sp, pop, s) : d5::launch_init(L, g, sp, pop, s);
}
inline cudaError_t launch_ga(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, int *dbg,
                             cudaStream_t s) {
    return L.sf == kScoreAD4 ? ad4::launch_ga(L, g, sp, pop, dbg, s) : d5::launch_ga(L, g, sp, pop, dbg, s);
}
inline cudaError_t launch_ls(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                             const LsArgs &a, int n_total, cudaStream_t s) {
    return L.sf == kScoreAD4 ? ad4::launch_ls(L, g, sp, pop, a, n_total, s)
                             : d5::launch_ls(L, g, sp, pop, a, n_total, s);
}
inline cudaError_t launch_bench_part(const LigDev &L, const GridDev &g, int part, int n, int iters,
                                     const float *genes, float *E, cudaStream_t s) {
    return L.sf == kScoreAD4 ? ad4::launch_bench_part(L, g, part, n, iters, genes, E, s)
                             : d5::launch_bench_part(L, g, part, n, iters, genes, E, s);
}
inline int adadelta_resident_groups(const LigDev &L) {
    return L.sf == kScoreAD4 ? ad4::adadelta_resident_groups(L) : d5::adadelta_resident_groups(L);
}
inline int run_sw_eligible(const LigDev &L, const SearchDev &sp) {
    return L.sf == kScoreAD4 ? ad4::run_sw_eligible(L, sp) : d5::run_sw_eligible(L, sp);
}
inline cudaError_t launch_run_sw(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                                 unsigned long long *prof, cudaStream_t s) {
    return L.sf == kScoreAD4 ? ad4::launch_run_sw(L, g, sp, pop, prof, s) : d5::launch_run_sw(L, g, sp, pop, prof, s);
}
inline cudaError_t launch_gen_end(const SearchDev &sp, const PopDev &pop, cudaStream_t s) {
    return d5::launch_gen_end(sp, pop, s);
}
inline cudaError_t launch_best(const LigDev &L, const SearchDev &sp, const PopDev &pop, float *bestE,
                               float *bestG, long long *evals, int *gens, cudaStream_t s) {
    return d5::launch_best(L, sp, pop, bestE, bestG, evals, gens, s);
}
inline cudaError_t launch_philox(int n, const uint32_t *ctr, const uint32_t *key, uint32_t *out, cudaStream_t s) {
    return d5::launch_philox(n, ctr, key, out, s);
}
inline cudaError_t launch_l2_gather(const float4 *buf, uint32_t n, int blocks, int iters, float *out, cudaStream_t s) {
    return d5::launch_l2_gather(buf, n, blocks, iters, out, s);
}
inline cudaError_t launch_stream_words(uint32_t k0, uint32_t k1, uint32_t purpose, uint32_t slot, uint32_t gen,
                                       uint32_t run, uint32_t m0, int n, uint32_t *out, cudaStream_t s) {
    return d5::launch_stream_words(k0, k1, purpose, slot, gen, run, m0, n, out, s);
}
#endif

}  // namespace dk
