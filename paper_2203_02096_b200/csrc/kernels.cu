// kernels.cu — sm_100a kernels of the LGA docking hot path.
//
//   k_init        a2   population init from Philox INIT words + energy (D8 gen 0)
//   k_ga          a9   elitism, tournaments, two-point crossover, mutation, offspring
//                      energy (D8); slot-0 group also draws the LS sample (a10)
//   k_ls_adadelta a7   fused persistent ADADELTA local search, energy + gradient every
//                      iteration, best tracking, Lamarckian writeback (D10)
//   k_ls_sw       a8   Solis-Wets; for small ligands both trial points x+b+d and x-b-d
//                      are scored at once by the two half-warps (speculative; the eval
//                      count still follows D9's sequential definition)
//   k_gen_end     a10  sum_evals (int64 warp reduction) + generation counter
//   k_best        a10  best-of-run argmin (lowest index on ties)
//   k_eval             parity hook / pose output: batched energy (+gradient, +pose)
//   k_philox, k_stream_words   parity hooks for D2
//
// Every kernel stages the per-ligand block ("cData") into shared memory; one lane
// group (16 or 32 lanes) handles one individual ("each local optimization occurs
// independently"; NS "one CTA or warp-group handles each individual").
#include <math.h>
#include <cstdlib>

#include <cooperative_groups.h>

#define DK_KERNELS_TU
#include "kernels.cuh"
#include "philox.cuh"
#include "score.cuh"

// This file is compiled once per (scoring function, part) in parallel (_build.py): the
// kernel templates are defined in every translation unit, but each part instantiates --
// launches -- only its own:
//   DK_PART 1  evaluation hooks, init, GA, generation end, best, microbenchmarks, RNG hooks
//   DK_PART 2  the ADADELTA local search (k_ls_adadelta)
//   DK_PART 3  the Solis-Wets local searches (k_ls_sw, k_ls_sw_tree, k_run_sw)
//   DK_PART 4  their parity-hook (TRACE) instantiations (dock_sw_trace)
// (one monolithic unit took ~5 min per scoring function to compile).
#ifndef DK_PART
#error "compile kernels.cu with -DDK_PART=1, 2, 3 or 4 (see _build.py)"
#endif

namespace dk {
namespace DK_SF_NS {   // d5, or ad4 when compiled with -DDK_AD4 (score.cuh)

// per-part pieces of launch_ls and setup_kernel_attributes (defined in parts 2 and 3)
cudaError_t launch_ls_adadelta(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                               const LsArgs &a, int n_total, cudaStream_t s);
cudaError_t launch_ls_sw(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                         const LsArgs &a, int n_total, cudaStream_t s);
cudaError_t setup_attributes_adadelta();
cudaError_t setup_attributes_sw();
template <bool TR>
cudaError_t launch_ls_sw_t(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                           const LsArgs &a, int n_total, cudaStream_t s);
cudaError_t setup_attributes_sw_trace();

static inline __host__ __device__ int a16(int x) { return (x + 15) & ~15; }

#if DK_PART == 1
ScratchLayout scratch_layout(const LigDev &L, bool grad, int extra) {
    ScratchLayout s;
    const int N = L.N, T = L.T, G = L.G;
    int o = 0;
    // the pair tiles (gradient kernels, and energy kernels of ligands too large for the
    // pair list, L.energy_tiles) keep the pose in the duplicated chunk layout [NC][2W]
    const bool dup = grad || L.energy_tiles;
    s.off_r = o; o += a16(dup ? 16 * 2 * L.Wg * L.NC : 16 * N);
    s.off_W = o; o += a16(48 * (T > 0 ? T : 1));
    s.off_tp = o; o += a16(4 * (T > 0 ? T : 1));
    // ts: back-projection rows (2N float4); packed tiles: also their pose rows (144 float4)
    // and the H-bond pair forces + per-atom totals (nhb + N <= 2N float4, prep.cpp)
    s.off_ts = o; if (grad) o += a16(32 * N > 16 * 144 || !L.packed ? 32 * N : 16 * 144);
    s.off_genes = o; o += a16(4 * G);
    s.off_grad = o; if (grad) o += a16(4 * G);
    s.off_extra = o; o += a16(extra);
    s.bytes = o;
    return s;
}

GroupCfg pick_group(int N) {
    GroupCfg c;
    if (N <= 16) { c.W = 16; c.MAXC = 1; return c; }
    c.W = 32;
    c.MAXC = N <= 32 ? 1 : (N <= 64 ? 2 : (N <= 96 ? 3 : (N <= 128 ? 4 : 8)));
    return c;
}
#endif

// Bytes of the ligand block a kernel stages: gradient kernels skip the pair list and the
// pair constants of the energy-only path.
static inline __host__ __device__ int staged_bytes(const LigDev &L, bool grad) {
    return (grad || L.energy_tiles) ? L.grad_bytes : L.blob_bytes;
}

__device__ __forceinline__ LigSm stage_ligand(const LigDev &L, uint8_t *sm, int bytes) {
    const uint4 *src = reinterpret_cast<const uint4 *>(L.blob);
    uint4 *dst = reinterpret_cast<uint4 *>(sm);
    for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    LigSm v;
    v.N = L.N; v.T = L.T; v.G = L.G; v.P = L.P; v.NW = L.NW; v.n_levels = L.n_levels;
    v.tlane = reinterpret_cast<const int *>(sm + L.off_tlane);
    v.tlane_top = L.tlane_top;
    v.p = reinterpret_cast<const float4 *>(sm + L.off_p);
    v.par = reinterpret_cast<const float4 *>(sm + L.off_par);
    v.meta = reinterpret_cast<const int *>(sm + L.off_meta);
    v.tA = reinterpret_cast<const float4 *>(sm + L.off_tA);
    v.tU = reinterpret_cast<const float4 *>(sm + L.off_tU);
    v.tmeta = reinterpret_cast<const int4 *>(sm + L.off_tmeta);
    v.pairs = reinterpret_cast<const uint32_t *>(sm + L.off_pairs);
    v.pprm = reinterpret_cast<const float4 *>(sm + L.off_pprm);
    v.mask = reinterpret_cast<const uint32_t *>(sm + L.off_mask);
    v.ppar = reinterpret_cast<const float4 *>(sm + L.off_ppar);
    v.NC = L.NC;
    v.tail_rot = L.tail_rot;
    v.tail_seg = L.tail_seg;
    v.slot_mode = L.slot_mode;
    v.slot4 = reinterpret_cast<const float4 *>(sm + L.off_slot4);
    v.slotq = reinterpret_cast<const float *>(sm + L.off_slotq);
    v.nhb = L.nhb;
    v.nhbr = L.nhbr;
    v.hbspan = L.hbspan;
    v.hbseg = reinterpret_cast<const int *>(sm + L.off_hbseg);
    v.hbc = reinterpret_cast<const float4 *>(sm + L.off_hbc);
    v.energy_tiles = L.energy_tiles;
    v.wA_v = L.wA_v; v.wB_v = L.wB_v; v.wA_h = L.wA_h; v.wB_h = L.wB_h; v.qscale = L.qscale;
    return v;
}

__device__ __forceinline__ Scratch scratch_at(uint8_t *base, const ScratchLayout &SL) {
    Scratch s;
    s.r = reinterpret_cast<float4 *>(base + SL.off_r);
    s.W = reinterpret_cast<float4 *>(base + SL.off_W);
    s.tp = reinterpret_cast<int *>(base + SL.off_tp);
    s.ts = reinterpret_cast<float4 *>(base + SL.off_ts);
    s.genes = reinterpret_cast<float *>(base + SL.off_genes);
    s.grad = reinterpret_cast<float *>(base + SL.off_grad);
    return s;
}

__device__ __forceinline__ bool run_active(const RunState &st, const SearchDev &sp) {
    return st.evals < sp.max_evals && st.gen < sp.max_generations;   // D8.5, checked per generation
}

__device__ __forceinline__ float nan_inf(float v) { return isnan(v) ? INFINITY : v; }

// ---------------------------------------------------------------------------
// k_eval: batched energy (+ gradient, + pose) of given genotypes.
// ---------------------------------------------------------------------------
template <int W, int MAXC, bool GRAD, int PARTS = kAll, bool PK = false>
__global__ void __launch_bounds__(256) k_eval(const LigDev L, const GridDev g, const ScratchLayout SL,
                                              int n, const float *__restrict__ genes, float *E,
                                              float *grad, float *xyz, const int *__restrict__ dfs2orig) {
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, GRAD));
    const int gl = threadIdx.x / W, sub = threadIdx.x % W;
    const int gi = blockIdx.x * (blockDim.x / W) + gl;
    if (gi >= n) return;
    const Scratch S = scratch_at(sm + staged_bytes(L, GRAD) + gl * SL.bytes, SL);
    const unsigned mask = group_mask<W>();
    const int G = L.G;
    for (int j = sub; j < G; j += W) S.genes[j] = genes[(size_t)gi * G + j];
    __syncwarp(mask);
    const float e = eval_group<W, MAXC, GRAD, PARTS, 1, PK>(Ls, g, S, sub, mask);
    if (sub == 0) E[gi] = e;
    if (GRAD && grad)
        for (int j = sub; j < G; j += W) grad[(size_t)gi * G + j] = S.grad[j];
    if (xyz) {
        for (int a = sub; a < L.N; a += W) {
            const float4 r = S.r[(GRAD || L.energy_tiles) ? ridx<W>(a) : a];
            float *o = xyz + ((size_t)gi * L.N + dfs2orig[a]) * 3;
            o[0] = r.x; o[1] = r.y; o[2] = r.z;
        }
    }
}

// ---------------------------------------------------------------------------
// k_init: generation 0 (D8): t uniform in the box, angles 2*pi*u01; evaluate.
// ---------------------------------------------------------------------------
template <int W, int MAXC>
__global__ void __launch_bounds__(256) k_init(const LigDev L, const GridDev g, const ScratchLayout SL,
                                              const SearchDev sp, const PopDev pop) {
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, false));
    const int gl = threadIdx.x / W, sub = threadIdx.x % W;
    const int gi = blockIdx.x * (blockDim.x / W) + gl;
    if (gi >= sp.runs * sp.pop) return;
    const int r = gi / sp.pop, k = gi % sp.pop, G = L.G;
    const Scratch S = scratch_at(sm + staged_bytes(L, false) + gl * SL.bytes, SL);
    const unsigned mask = group_mask<W>();
    const uint2 key = make_uint2(sp.key0, sp.key1);
    const uint32_t run_g = (uint32_t)(sp.run_base + r);
    float *row = pop.genes + ((size_t)r * sp.pop + k) * G;          // buffer 0 (generation 0)
    for (int j = sub; j < G; j += W) {
        const float u = u01(stream_word(key, kInit, (uint32_t)k, 0u, run_g, (uint32_t)j));
        float v;
        if (j == 0) v = g.ox + u * (g.hx - g.ox);
        else if (j == 1) v = g.oy + u * (g.hy - g.oy);
        else if (j == 2) v = g.oz + u * (g.hz - g.oz);
        else v = 6.28318530717958647692f * u;
        S.genes[j] = v;
        row[j] = v;
    }
    __syncwarp(mask);
    const float e = eval_group<W, MAXC, false>(Ls, g, S, sub, mask);
    if (sub == 0) {
        pop.E[(size_t)r * sp.pop + k] = e;
        if (k == 0) { pop.state[r].evals = sp.pop; pop.state[r].gen = 0; pop.ls_count[r] = 0; }
    }
}

// D8 tournament between two distinct candidates (ties -> lower index, NaN = +inf).
__device__ __forceinline__ int tournament(const float *E, int pop, uint32_t wa, uint32_t wb, uint32_t wc,
                                          float p_tour) {
    const int i = (int)below(wa, (uint32_t)pop);
    int j = (int)below(wb, (uint32_t)(pop - 1));
    if (j >= i) j += 1;
    const float ei = nan_inf(__ldcg(E + i)), ej = nan_inf(__ldcg(E + j));   // L2: written by other CTAs (k_run_sw)
    const int better = (ei < ej || (ei == ej && i < j)) ? i : j;
    const int other = better == i ? j : i;
    return u01(wc) < p_tour ? better : other;
}

// ---------------------------------------------------------------------------
// k_ga: one generation of the GA for every (run, slot) (D8).
// ---------------------------------------------------------------------------
// One GA slot (D8) of run r, generation st.gen + 1, on one lane group: slot 0 =
// elitism + the LS sample (partial Fisher-Yates), slot k >= 1 = tournaments, two-point
// crossover, mutation and the offspring energy.  act = false: a shadow evaluation of a
// dummy genotype keeps the warp converged and writes nothing.  Used by k_ga (one launch
// per generation) and by k_run_sw (the persistent cluster kernel).
template <int W, int MAXC>
__device__ __forceinline__ void ga_slot_group(const LigSm &Ls, const GridDev &g, const Scratch &S, int *perm_scratch,
                                              const SearchDev &sp, const PopDev &pop, const int G, bool act,
                                              const RunState st, int r, int k, int sub, int *dbg) {
    const int P = sp.pop;
    const unsigned mask = group_mask<W>();
    const uint2 key = make_uint2(sp.key0, sp.key1);
    const uint32_t gen = act ? (uint32_t)st.gen + 1u : 1u;
    const int cur = act ? (st.gen & 1) : 0, nxt = gen & 1;
    const int rr = act ? r : 0;
    const float *oldG = pop.genes + ((size_t)cur * sp.rstride + rr) * P * G;
    const float *oldE = pop.E + ((size_t)cur * sp.rstride + rr) * P;
    float *newG = pop.genes + ((size_t)nxt * sp.rstride + rr) * P * G;
    float *newE = pop.E + ((size_t)nxt * sp.rstride + rr) * P;
    const uint32_t run_g = (uint32_t)(sp.run_base + rr);
    bool child = false;                 // this group scores a real offspring
    int A = 0, B = 0, c1 = 0, c2 = 0;
    bool cross = false;
    unsigned long long mbits = 0ull;

    if (!act) {
        for (int j = sub; j < G; j += W) S.genes[j] = 0.0f;
    } else if (k == 0) {
        // elitism: argmin, NaN = +inf, ties -> lowest index; copied without re-evaluation
        float bv = INFINITY;
        int bi = 0x7fffffff;
        for (int i = sub; i < P; i += W) {
            const float v = nan_inf(__ldcg(oldE + i));
            if (v < bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
#pragma unroll
        for (int m = W / 2; m >= 1; m >>= 1) {
            const float ov = __shfl_xor_sync(mask, bv, m, W);
            const int oi = __shfl_xor_sync(mask, bi, m, W);
            if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        for (int j = sub; j < G; j += W) {
            const float v = __ldcg(oldG + (size_t)bi * G + j);
            newG[j] = v;
            S.genes[j] = v;                 // shadow evaluation only
        }
        if (sub == 0) newE[0] = __ldcg(oldE + bi);
        // local-search sample: partial Fisher-Yates over the new population (D8.3)
        int *perm = perm_scratch;
        for (int i = sub; i < P; i += W) perm[i] = i;
        __syncwarp(mask);
        if (sub == 0) {
            uint4 blk = make_uint4(0, 0, 0, 0);
            for (int s = 0; s < sp.n_ls; ++s) {
                if ((s & 3) == 0) blk = stream_block(key, kLsPick, 0u, gen, run_g, (uint32_t)(s >> 2));
                const int j = s + (int)below(lane_of(blk, s & 3), (uint32_t)(P - s));
                const int t = perm[s]; perm[s] = perm[j]; perm[j] = t;
            }
        }
        __syncwarp(mask);
        for (int s = sub; s < P; s += W) pop.perm[(size_t)r * P + s] = perm[s];
        if (dbg && sub == 0) {
            int *d = dbg + (size_t)(r * P + k) * 8;
            d[0] = bi; d[1] = bi; d[2] = 0; d[3] = 0; d[4] = 0; d[5] = 0; d[6] = 0; d[7] = bi;
        }
    } else {
        // slot k >= 1: words 0..8 from the first three Philox blocks
        child = true;
        const uint4 b0 = stream_block(key, kGA, (uint32_t)k, gen, run_g, 0u);
        const uint4 b1 = stream_block(key, kGA, (uint32_t)k, gen, run_g, 1u);
        const uint4 b2 = stream_block(key, kGA, (uint32_t)k, gen, run_g, 2u);
        A = tournament(oldE, P, b0.x, b0.y, b0.z, sp.p_tour);
        B = tournament(oldE, P, b0.w, b1.x, b1.y, sp.p_tour);
        cross = u01(b1.z) < sp.p_cross;
        if (cross) {
            c1 = (int)below(b1.w, (uint32_t)(G + 1));
            c2 = (int)below(b2.x, (uint32_t)(G + 1));
            if (c2 < c1) { const int t = c1; c1 = c2; c2 = t; }
        }
        for (int j = sub; j < G; j += W) {
            const uint32_t m = 9u + 2u * (uint32_t)j;                 // mutation coin; delta = m + 1
            const uint4 bc = stream_block(key, kGA, (uint32_t)k, gen, run_g, m >> 2);
            const uint32_t wc = lane_of(bc, m & 3);
            const uint32_t md = m + 1u;
            const uint32_t wd = ((md >> 2) == (m >> 2)) ? lane_of(bc, md & 3)
                                                        : lane_of(stream_block(key, kGA, (uint32_t)k, gen, run_g, md >> 2), md & 3);
            float v = __ldcg(oldG + (size_t)((cross && c1 <= j && j < c2) ? B : A) * G + j);
            if (u01(wc) < sp.p_mut) {
                const float mag = j < 3 ? sp.mut_trans : sp.mut_angle;
                v += (2.0f * u01(wd) - 1.0f) * mag;
                mbits |= 1ull << j;
            }
            S.genes[j] = v;
        }
    }
    __syncwarp();
    const float e = eval_group<W, MAXC, false>(Ls, g, S, sub, 0xffffffffu);
    if (!child) return;
    for (int j = sub; j < G; j += W) newG[(size_t)k * G + j] = S.genes[j];
    if (sub == 0) newE[k] = e;
    if (dbg) {
#pragma unroll
        for (int m = W / 2; m >= 1; m >>= 1) mbits |= __shfl_xor_sync(mask, mbits, m, W);
        if (sub == 0) {
            int *d = dbg + (size_t)(r * P + k) * 8;
            d[0] = A; d[1] = B; d[2] = cross ? 1 : 0; d[3] = c1; d[4] = c2;
            d[5] = (int)(uint32_t)mbits; d[6] = (int)(uint32_t)(mbits >> 32); d[7] = -1;
        }
    }
}

// ---------------------------------------------------------------------------
// k_ga: one generation of the GA for every (run, slot) (D8).
// ---------------------------------------------------------------------------
template <int W, int MAXC>
__global__ void __launch_bounds__(256) k_ga(const LigDev L, const GridDev g, const ScratchLayout SL,
                                            const SearchDev sp, const PopDev pop, int *dbg) {
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int gl = threadIdx.x / W, sub = threadIdx.x % W;
    const int gi = blockIdx.x * (blockDim.x / W) + gl;
    const int P = sp.pop, G = L.G;
    bool act = false;
    RunState st;
    const int r = gi / P;
    if (gi < sp.runs * P) { st = pop.state[r]; act = run_active(st, sp); }
    if (!__syncthreads_or(act)) return;            // finished runs cost one state read
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, false));
    // Both lane groups of a warp stay converged through the evaluation (the elite slot and
    // inactive groups evaluate a dummy genotype and write nothing), so its shuffles take a
    // constant full-warp mask.
    if (!__any_sync(0xffffffffu, act)) return;
    uint8_t *gbase = sm + staged_bytes(L, false) + gl * SL.bytes;
    ga_slot_group<W, MAXC>(Ls, g, scratch_at(gbase, SL), reinterpret_cast<int *>(gbase + SL.off_extra), sp, pop, G,
                           act, st, r, gi % P, sub, dbg);
}

// Resolve the row a local-search group works on (engine or hook mode).
struct LsTarget {
    bool act;
    float *row;
    float *E;
    int *evals;
    uint32_t slot, gen, run_g;
    int run_l;                    // engine mode: run index in the launch (for the fused gen end); -1: hook
    int idx;                      // hook mode: index of the individual in the call (fed / trace rows); -1: engine
};

__device__ __forceinline__ LsTarget ls_target(const SearchDev &sp, const PopDev &pop, const LsArgs &a, int gi,
                                              int G) {
    LsTarget t;
    t.act = false;
    t.run_l = -1;
    t.idx = -1;
    if (a.use_state) {
        if (gi >= sp.runs * a.n_per_run) return t;
        const int r = gi / a.n_per_run, s = gi % a.n_per_run;
        RunState st;
        st.evals = __ldcg(&pop.state[r].evals); st.gen = __ldcg(&pop.state[r].gen);   // L2: k_run_sw
        if (!run_active(st, sp)) return t;
        const int gen = st.gen + 1, nxt = gen & 1;
        const int i = __ldcg(pop.perm + (size_t)r * sp.pop + s);
        t.row = pop.genes + (((size_t)nxt * sp.rstride + r) * sp.pop + i) * G;
        t.E = pop.E + ((size_t)nxt * sp.rstride + r) * sp.pop + i;
        t.evals = pop.ls_evals + (size_t)r * sp.pop + s;
        t.slot = (uint32_t)i; t.gen = (uint32_t)gen; t.run_g = (uint32_t)(sp.run_base + r);
        t.run_l = r;
        t.act = true;
    } else {
        if (gi >= a.n_per_run) return t;
        t.row = a.genes + (size_t)gi * G;
        t.E = a.E + gi;
        t.evals = a.evals + gi;
        t.slot = (uint32_t)a.rng_slot[gi]; t.gen = (uint32_t)a.gen; t.run_g = (uint32_t)a.run;
        t.idx = gi;
        t.act = true;
    }
    return t;
}

// Generation end fused into the LS kernels (D11 sum_evals, and the generation
// counter; formerly the k_gen_end launch): every LS individual of a run bumps the run's
// counter after writing its evaluation count, and the run's last one (classic last-block
// pattern) sums the counts and advances the run state.  Integer sum: order-free, so the
// result equals k_gen_end's.
__device__ __forceinline__ void ls_finish(const SearchDev &sp, const PopDev &pop, const LsTarget &t) {
    if (t.run_l < 0) return;
    const int r = t.run_l;
    __threadfence();
    if (atomicAdd(&pop.ls_count[r], 1) != sp.n_ls - 1) return;
    __threadfence();
    long long s = 0;
    for (int i = 0; i < sp.n_ls; ++i) s += __ldcg(pop.ls_evals + (size_t)r * sp.pop + i);
    const long long ev = __ldcg(&pop.state[r].evals);
    const int gen = __ldcg(&pop.state[r].gen);
    pop.state[r].evals = ev + (long long)(sp.pop - 1) + s;   // offspring + local search
    pop.state[r].gen = gen + 1;
    pop.ls_count[r] = 0;
}

// ---------------------------------------------------------------------------
// k_ls_adadelta: max_iters x (energy + gradient, ADADELTA step), best tracking (D10).
// ---------------------------------------------------------------------------
#ifndef DK_ADA_MINB
#define DK_ADA_MINB 2   // min resident CTAs/SM for the ADADELTA kernel (register cap 65536/(256*MINB))
#endif
// TRACE: the parity-hook instantiation (dock_ad_trace: fed inputs and traces, LsArgs::ad_*);
// the production instantiation carries none of that code (register pressure at the cap).
template <int W, int MAXC, bool TRACE = false, bool PK = false>
__global__ void __launch_bounds__(256, (MAXC <= 4 ? DK_ADA_MINB : 1)) k_ls_adadelta(const LigDev L, const GridDev g, const ScratchLayout SL,
                                                     const SearchDev sp, const PopDev pop, const LsArgs a) {
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int gl = threadIdx.x / W, sub = threadIdx.x % W;
    const int gi = blockIdx.x * (blockDim.x / W) + gl;
    const int G = L.G;
    const LsTarget t = ls_target(sp, pop, a, gi, G);
    if (!__syncthreads_or(t.act)) return;
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, true));
    // Both lane groups of a warp stay converged (an inactive group shadows its partner on a
    // dummy genotype and writes nothing), so the group shuffles take a constant full-warp
    // mask: no divergence checks around every SHFL (measured: MATCH.ANY + BRA.DIV paths).
    if (!__any_sync(0xffffffffu, t.act)) return;
    const Scratch S = scratch_at(sm + staged_bytes(L, true) + gl * SL.bytes, SL);
    constexpr unsigned mask = 0xffffffffu;
    // genes per lane: the packed variant is only chosen for G <= 32 (prep.cpp), one per lane
    constexpr int NSET = PK ? 1 : (kMaxGenes + W - 1) / W;
    float x[NSET], sg[NSET], sd[NSET], bx[NSET];
#pragma unroll
    for (int s = 0; s < NSET; ++s) {
        const int j = sub + W * s;
        x[s] = (j < G && t.act) ? t.row[j] : 0.0f;
        bx[s] = x[s]; sg[s] = 0.0f; sd[s] = 0.0f;
        if (j < G) S.genes[j] = x[s];
    }
    float Ebest = t.act ? *t.E : 0.0f;
    const float rho = sp.ad_rho, eps = sp.ad_eps;
    __syncwarp(mask);
    for (int it = 0; it < a.iters; ++it) {
        float E = eval_group<W, MAXC, true, kAll, 1, PK>(Ls, g, S, sub, mask);
        if constexpr (TRACE) {            // parity hook only
            const size_t row = (size_t)t.idx * a.iters + it;
            if (a.ad_fed && t.act) {
                E = a.ad_fed[row * (G + 1)];
                for (int j = sub; j < G; j += W) S.grad[j] = a.ad_fed[row * (G + 1) + 1 + j];
            }
            __syncwarp(mask);
            if (a.ad_trace_x && t.act) {
#pragma unroll
                for (int s = 0; s < NSET; ++s) {
                    const int j = sub + W * s;
                    if (j < G) { a.ad_trace_x[row * G + j] = x[s]; a.ad_trace_g[row * G + j] = S.grad[j]; }
                }
                if (sub == 0) a.ad_trace_E[row] = E;
            }
        }
        if (E < Ebest) {
            Ebest = E;
#pragma unroll
            for (int s = 0; s < NSET; ++s) bx[s] = x[s];
        }
#pragma unroll
        for (int s = 0; s < NSET; ++s) {
            const int j = sub + W * s;
            if (j < G) {
                const float gj = S.grad[j];
                sg[s] = rho * sg[s] + (1.0f - rho) * gj * gj;
                const float dx = -sqrtf(sd[s] + eps) * rsqrtf(sg[s] + eps) * gj;
                sd[s] = rho * sd[s] + (1.0f - rho) * dx * dx;
                x[s] += dx;
                S.genes[j] = x[s];
            }
        }
        __syncwarp(mask);
    }
    if (!t.act) return;
#pragma unroll
    for (int s = 0; s < NSET; ++s) {
        const int j = sub + W * s;
        if (j < G) t.row[j] = bx[s];
    }
    if (sub == 0) { *t.E = Ebest; *t.evals = a.iters; ls_finish(sp, pop, t); }
}

// ---------------------------------------------------------------------------
// Solis-Wets arithmetic (D9), written with explicit round-to-nearest intrinsics so every
// kernel that replays it (k_ls_sw, the speculative k_ls_sw_tree, its resolution step)
// produces bit-identical genes: no FMA contraction can differ between call sites.
// ---------------------------------------------------------------------------
// (u1 - 1/2) + (u2 - 1/2) of gene j, iteration it: state independent (counter-based, D2)
__device__ __forceinline__ float sw_tri(const uint2 key, uint32_t slot, uint32_t gen, uint32_t run, int G, int it,
                                        int j) {
    const uint32_t m = 2u * (uint32_t)G * (uint32_t)it + 2u * (uint32_t)j;   // m even: m, m+1 share a block
    const uint4 blk = stream_block(key, kSW, slot, gen, run, m >> 2);
    const uint32_t w1 = lane_of(blk, m & 3), w2 = lane_of(blk, (m + 1) & 3);
    return __fadd_rn(u01(w1) - 0.5f, u01(w2) - 0.5f);
}
// d = rho * tri: the centred triangular deviate on (-rho, rho) (exact in FP32)
__device__ __forceinline__ float sw_dev(float rho, float tri) { return __fmul_rn(rho, tri); }
__device__ __forceinline__ float sw_deviate(const uint2 key, uint32_t slot, uint32_t gen, uint32_t run, int G, int it,
                                            int j, float rho) {
    return sw_dev(rho, sw_tri(key, slot, gen, run, G, it, j));
}
__device__ __forceinline__ float sw_c1(float x, float b, float d) { return __fadd_rn(__fadd_rn(x, b), d); }
__device__ __forceinline__ float sw_c2(float x, float b, float d) { return __fsub_rn(__fsub_rn(x, b), d); }
// outcome o: 0 = x+b+d accepted, 1 = x-b-d accepted, 2 = both rejected
__device__ __forceinline__ void sw_gene_step(int o, float d, float &x, float &b) {
    if (o == 0) { x = sw_c1(x, b, d); b = __fmaf_rn(0.2f, b, __fmul_rn(0.4f, d)); }
    else if (o == 1) { x = sw_c2(x, b, d); b = __fsub_rn(b, __fmul_rn(0.4f, d)); }
    else { b = __fmul_rn(0.5f, b); }
}
__device__ __forceinline__ void sw_scalar_step(int o, const SearchDev &sp, float &rho, int &succ, int &fail) {
    if (o < 2) { ++succ; fail = 0; } else { ++fail; succ = 0; }
    if (succ >= sp.sw_cons_succ) { rho *= sp.sw_expand; succ = 0; }
    if (fail >= sp.sw_cons_fail) { rho *= sp.sw_contract; fail = 0; }
}

// ---------------------------------------------------------------------------
// k_ls_sw: Solis-Wets (D9; P:64 citing Solis & Wets 1981).  One warp per individual.
// W <= 16: the two half-warps score x+b+d and x-b-d concurrently.
// ---------------------------------------------------------------------------
// TRACE: the parity-hook instantiation (dock_sw_trace: fed energies, outcome traces).
template <int W, int MAXC, bool TRACE = false>
__global__ void __launch_bounds__(256) k_ls_sw(const LigDev L, const GridDev g, const ScratchLayout SL,
                                               const SearchDev sp, const PopDev pop, const LsArgs a) {
    constexpr int NG = (W <= 16) ? 2 : 1;
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / W, sub = lane % W;
    const int wi = blockIdx.x * (blockDim.x >> 5) + warp;
    const int G = L.G;
    const LsTarget t = ls_target(sp, pop, a, wi, G);
    if (!__syncthreads_or(t.act)) return;
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, false));
    if (!t.act) return;
    uint8_t *wbase = sm + staged_bytes(L, false) + (size_t)warp * NG * SL.bytes;
    const Scratch S0 = scratch_at(wbase, SL);
    const Scratch S1 = scratch_at(wbase + (NG - 1) * SL.bytes, SL);
    const Scratch Sg = grp == 0 ? S0 : S1;
    constexpr unsigned gmask = 0xffffffffu;   // a warp = one individual: both groups always converged
    const uint2 key = make_uint2(sp.key0, sp.key1);
    constexpr int NSET = (kMaxGenes + 31) / 32;
    float x[NSET], b[NSET], d[NSET], c1[NSET], c2[NSET];
#pragma unroll
    for (int s = 0; s < NSET; ++s) {
        const int j = lane + 32 * s;
        x[s] = j < G ? t.row[j] : 0.0f;
        b[s] = 0.0f; d[s] = 0.0f; c1[s] = 0.0f; c2[s] = 0.0f;
    }
    float Ex = *t.E;
    float rho = sp.sw_rho;
    int succ = 0, fail = 0, ne = 0;
    for (int it = 0; it < a.iters; ++it) {
        if (rho < sp.sw_rho_min) break;
#pragma unroll
        for (int s = 0; s < NSET; ++s) {
            const int j = lane + 32 * s;
            if (j < G) {
                d[s] = sw_deviate(key, t.slot, t.gen, t.run_g, G, it, j, rho);
                c1[s] = sw_c1(x[s], b[s], d[s]);
                c2[s] = sw_c2(x[s], b[s], d[s]);
                S0.genes[j] = c1[s];
                if (NG == 2) S1.genes[j] = c2[s];
            }
        }
        __syncwarp();
        float E1, E2 = 0.0f;
        const float *fed = (TRACE && a.sw_fed) ? a.sw_fed + ((size_t)t.idx * a.iters + it) * 2 : nullptr;   // parity mode
        if (NG == 2) {
            const float e = eval_group<W, MAXC, false>(Ls, g, Sg, sub, gmask);
            E1 = __shfl_sync(0xffffffffu, e, 0);
            E2 = __shfl_sync(0xffffffffu, e, W);
            if constexpr (TRACE) if (fed) { E1 = fed[0]; E2 = fed[1]; }
        } else {
            // x+b+d, then x-b-d only if the first failed: one evaluation call site (the
            // kernel's instruction footprint matters at one warp per SM)
            E1 = INFINITY;
            for (int trial = 0; trial < 2; ++trial) {
                if (trial == 1) {
                    if (E1 < Ex) break;
                    __syncwarp();
#pragma unroll
                    for (int s = 0; s < NSET; ++s) {
                        const int j = lane + 32 * s;
                        if (j < G) S0.genes[j] = c2[s];
                    }
                    __syncwarp();
                }
                float e = eval_group<W, MAXC, false>(Ls, g, S0, sub, gmask);
                if constexpr (TRACE) if (fed) e = fed[trial];
                if (trial == 0) E1 = e; else E2 = e;
            }
        }
        const float rho_it = rho;
        int o;
        ++ne;
        if (E1 < Ex) {
#pragma unroll
            for (int s = 0; s < NSET; ++s) sw_gene_step(0, d[s], x[s], b[s]);
            Ex = E1;
            o = 0;
        } else {
            ++ne;
            if (E2 < Ex) {
#pragma unroll
                for (int s = 0; s < NSET; ++s) sw_gene_step(1, d[s], x[s], b[s]);
                Ex = E2;
                o = 1;
            } else {
#pragma unroll
                for (int s = 0; s < NSET; ++s) sw_gene_step(2, d[s], x[s], b[s]);
                o = 2;
            }
        }
        sw_scalar_step(o, sp, rho, succ, fail);
        if constexpr (TRACE) if (lane == 0) {
            a.sw_trace[(size_t)t.idx * a.iters + it] = o;
            a.sw_trace_rho[(size_t)t.idx * a.iters + it] = rho_it;
        }
        __syncwarp();
    }
#pragma unroll
    for (int s = 0; s < NSET; ++s) {
        const int j = lane + 32 * s;
        if (j < G) t.row[j] = x[s];
    }
    if (lane == 0) { *t.E = Ex; *t.evals = ne; ls_finish(sp, pop, t); }
}

// ---------------------------------------------------------------------------
// k_ls_sw_tree: speculative Solis-Wets for under-filled launches (1stp: 9 LS individuals
// x 20 runs = 180 chains on 148 SMs).  Each SW iteration has three outcomes (x+b+d
// accepted, x-b-d accepted, both rejected, D9), and the next iteration's deviates are
// known in advance (counter-based Philox, D2).  So one CTA of 3^D - 1 lane groups
// evaluates every trial point of the next D iterations at once: level l holds 3^l parent
// states x 2 candidates.  Afterwards the actual path is resolved sequentially from the
// energies, with exactly D9's decisions and evaluation count.  Every group replays its
// path with the same sw_* arithmetic as the resolution, so the result is bit-identical
// to k_ls_sw; only the latency changes (D iterations per evaluation round trip).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ipow3(int d) { return d == 0 ? 1 : 3 * ipow3(d - 1); }
template <int W, int D, int KP = 1>
constexpr int tree_threads() { return ((ipow3(D) - 1) * KP * W + 31) / 32 * 32; }

// KP > 1: every node is evaluated cooperatively by KP lane groups (large ligands, whose
// single evaluation is the latency of the chain): each computes a part of the grid and
// pair sums, the partials are added in a fixed order in the resolution step.
// The speculative Solis-Wets chain of one individual (t) on one CTA of (3^D - 1) * KP lane
// groups, ligand already staged (k_ls_sw_tree, and the LS phase of k_run_sw).  Shared
// memory after the ligand block: the groups' scratch, then x, b, partial energies and the
// double-buffered deviate shapes (tree_smem).
#ifndef DK_TRI_AHEAD
#define DK_TRI_AHEAD 32
#endif
constexpr int kTriAhead = DK_TRI_AHEAD;   // SW iterations whose deviate shapes are precomputed at a time (>= D)

template <int W, int MAXC, int D, int KP, bool TRACE = false>
__device__ __forceinline__ void sw_tree_chain(const LigSm &Ls, const GridDev &g, const ScratchLayout &SL,
                                              const SearchDev &sp, const PopDev &pop, const LsArgs &a,
                                              const LsTarget &t, uint8_t *sm, const int staged, const int G) {
    constexpr int NGR = ipow3(D) - 1;
    constexpr int NS = (kMaxGenes + W - 1) / W;              // genes per lane: j = sub + W s
    float *sE = reinterpret_cast<float *>(sm + staged + NGR * KP * SL.bytes);   // [2][NGR][KP], by round parity
    float *stri = sE + 2 * NGR * KP;                         // [kTriAhead][G] deviate shapes of iterations sbase..
    const int gidx = threadIdx.x / W, sub = threadIdx.x % W;  // lane group
    const int grp = gidx / KP, part = gidx % KP;             // node, part of its evaluation
    const bool in_grp = grp < NGR;
    const Scratch S = scratch_at(sm + staged + (in_grp ? gidx : 0) * SL.bytes, SL);
    // every group evaluates every round (a moot node on stale genes, result unused), so
    // the warps stay converged and the group shuffles take a constant full-warp mask
    constexpr unsigned gmask = 0xffffffffu;
    const uint2 key = make_uint2(sp.key0, sp.key1);
    // x and b live in registers: every thread holds genes sub + W s and advances them along
    // the resolved path itself (all threads resolve identically), so a round needs one
    // barrier; sE is double-buffered by round parity for the same reason.
    float x[NS], b[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
        const int j = sub + W * s2;
        x[s2] = j < G ? __ldcg(t.row + j) : 0.0f;
        b[s2] = 0.0f;
    }
    for (int j = sub; j < G; j += W) S.genes[j] = 0.0f;      // finite genes for a moot first round
    // this group's node: level lvl, parent state sigma (base-3 outcome digits), candidate
    int lvl = 0;
    while (lvl + 1 < D && grp >= ipow3(lvl + 1) - 1) ++lvl;
    const int sigma = (grp - (ipow3(lvl) - 1)) >> 1, cand = (grp - (ipow3(lvl) - 1)) & 1;
    int digit[D];
    {
        int v = sigma;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) {
            digit[k] = 0;
            if (k < lvl) { digit[k] = v % 3; v /= 3; }
        }
    }
    // deviate shapes of kTriAhead iterations at a time (one Philox block per (iteration,
    // gene)), refilled when a round would run past them: the Philox work leaves the
    // per-round critical path
    // (only the iterations the chain can still reach: min(kTriAhead, iters - sbase); a node
    // beyond a.iters is never live, so the unfilled tail of the window is never read)
    int sbase = 0;
    for (int q = threadIdx.x; q < min(kTriAhead, a.iters) * G; q += blockDim.x) {
        const int k = q / G, j = q - k * G;
        stri[q] = sw_tri(key, t.slot, t.gen, t.run_g, G, k, j);
    }
    __syncthreads();
    float Ex = __ldcg(t.E), rho = sp.sw_rho;
    int succ = 0, fail = 0, ne = 0, it = 0, cur = 0;
    while (it < a.iters && !(rho < sp.sw_rho_min)) {
        if (it + D > sbase + kTriAhead) {                     // uniform: refill the deviate window
            __syncthreads();                                  // the previous round's path reads are done
            sbase = it;
            for (int q = threadIdx.x; q < min(kTriAhead, a.iters - sbase) * G; q += blockDim.x) {
                const int k = q / G, j = q - k * G;
                stri[q] = sw_tri(key, t.slot, t.gen, t.run_g, G, sbase + k, j);
            }
            __syncthreads();
        }
        const float *tri = stri + (it - sbase) * G;           // iteration it + k: tri[k * G + j]
        float *sEc = sE + cur * NGR * KP;
        // ---- 1. every live node's trial genotype, then its energy ----
        if (in_grp) {
            float rl[D];
            float r = rho;
            int su = succ, fa = fail;
            bool live = true;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                rl[k] = r;
                if (k < lvl) {
                    if (r < sp.sw_rho_min) live = false;
                    sw_scalar_step(digit[k], sp, r, su, fa);
                }
            }
            if (r < sp.sw_rho_min || it + lvl >= a.iters) live = false;
            if (live) {
#pragma unroll
                for (int s2 = 0; s2 < NS; ++s2) {
                    const int j = sub + W * s2;
                    if (j < G) {
                        float xx = x[s2], bb = b[s2];
#pragma unroll
                        for (int k = 0; k < D; ++k)
                            if (k < lvl) sw_gene_step(digit[k], sw_dev(rl[k], tri[k * G + j]), xx, bb);
                        const float d = sw_dev(r, tri[lvl * G + j]);
                        S.genes[j] = cand ? sw_c2(xx, bb, d) : sw_c1(xx, bb, d);
                    }
                }
            }
            __syncwarp(gmask);
            float e = eval_group<W, MAXC, false, kAll, KP>(Ls, g, S, sub, gmask, part);
            if constexpr (TRACE)                                   // parity mode: the fed energy
                if (a.sw_fed && live) e = part == 0 ? a.sw_fed[((size_t)t.idx * a.iters + it + lvl) * 2 + cand] : 0.0f;
            if (sub == 0) sEc[gidx] = live ? e : INFINITY;
        }
        __syncthreads();
        // ---- 2. resolve the actual path (every thread, identical scalar logic) ----
        int path[D], rho_steps = 0;
        float rl[D];
        int sg = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            path[k] = 2; rl[k] = 0.0f;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (it >= a.iters || rho < sp.sw_rho_min) break;
            rl[k] = rho;
            const int id = ipow3(k) - 1 + 2 * sg;
            float E1 = sEc[id * KP], E2 = sEc[(id + 1) * KP];          // partials: fixed order
#pragma unroll
            for (int p = 1; p < KP; ++p) { E1 += sEc[id * KP + p]; E2 += sEc[(id + 1) * KP + p]; }
            int o;
            ++ne;
            if (E1 < Ex) { o = 0; Ex = E1; }
            else {
                ++ne;
                if (E2 < Ex) { o = 1; Ex = E2; }
                else o = 2;
            }
            sw_scalar_step(o, sp, rho, succ, fail);
            if constexpr (TRACE) if (threadIdx.x == 0) {
                a.sw_trace[(size_t)t.idx * a.iters + it] = o;
                a.sw_trace_rho[(size_t)t.idx * a.iters + it] = rl[k];
            }
            path[k] = o;
            sg = 3 * sg + o;
            ++it;
            ++rho_steps;
        }
        // ---- 3. advance this thread's x and b along the resolved path ----
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
            const int j = sub + W * s2;
            if (j < G) {
#pragma unroll
                for (int k = 0; k < D; ++k)
                    if (k < rho_steps) sw_gene_step(path[k], sw_dev(rl[k], tri[k * G + j]), x[s2], b[s2]);
            }
        }
        cur ^= 1;
    }
    if (gidx == 0) {
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
            const int j = sub + W * s2;
            if (j < G) t.row[j] = x[s2];
        }
    }
    if (threadIdx.x == 0) { *t.E = Ex; *t.evals = ne; ls_finish(sp, pop, t); }
}

template <int W, int MAXC, int D, int KP = 1, bool TRACE = false>
__global__ void __launch_bounds__(tree_threads<W, D, KP>(), (W == 16 && D == 3) ? 2 : 1) k_ls_sw_tree(const LigDev L, const GridDev g,
                                                                     const ScratchLayout SL, const SearchDev sp,
                                                                     const PopDev pop, const LsArgs a) {
    constexpr int NGR = ipow3(D) - 1;
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int G = L.G;
    const LsTarget t = ls_target(sp, pop, a, blockIdx.x, G);
    if (!t.act) return;                                      // uniform: one individual per CTA
    const int staged = staged_bytes(L, false);
    const LigSm Ls = stage_ligand(L, sm, staged);
    sw_tree_chain<W, MAXC, D, KP, TRACE>(Ls, g, SL, sp, pop, a, t, sm, staged, G);
}

// ---------------------------------------------------------------------------
// k_run_sw: a whole Solis-Wets docking run per thread-block cluster, persistent over its
// generations.  One cluster of n_ls CTAs per run (n_ls <= 16: non-portable
// cluster size); CTA q of the cluster owns the run's q-th LS individual.  Per generation:
//   GA phase: the cluster's n_ls x 8 lane groups deal the pop GA slots (ga_slot_group: the
//     same per-slot arithmetic and Philox words as k_ga), cluster barrier;
//   LS phase: every CTA runs its individual's speculative depth-2 chain (sw_tree_chain),
//     the run's last chain advances the run state (ls_finish), cluster barrier;
// until the run's budget is spent (D8.5 per run, on the device).  Results equal the
// lockstep and branched engines'.  No launch, graph node or host poll per generation, and
// no run waits for another run's chains.  Population data written by other CTAs of the
// cluster is read through L2 (__ldcg); the barriers order it (release / acquire).
// prof != null: CTA 0 of run 0 accumulates the LS-phase duration (GA barrier -> LS
// barrier, %globaltimer ns) and the phase count.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Extra warps per k_run_sw CTA that work only in the GA phase: with
// n_ls x (3^D - 1) lane groups the 1stp cluster (9 x 8 groups) deals its 150 GA slots in
// 3 rounds, with one more warp (9 x 10 groups) in 2.  In the LS phase they are idle
// (not in the tree).  Their scratch overlaps the tree's sE / deviate window, which only
// the LS phase uses; the cluster barriers separate the phases.
#ifndef DK_RUNSW_XWARPS
#define DK_RUNSW_XWARPS 0
#endif
#ifndef DK_RUNSW_SPEC
#define DK_RUNSW_SPEC 0   // 1: speculative GA slots in the LS phase (A/B: 1stp 0.99x, PS 0.96x -- DESIGN.md §15)
#endif
template <int W, int D>
__host__ __device__ constexpr int run_sw_threads() { return tree_threads<W, D, 1>() + 32 * DK_RUNSW_XWARPS; }

template <int W, int MAXC, int D = 2>
#if DK_RUNSW_XWARPS > 0
// 2 CTAs of 5 warps per SM need <= 3 warps per SM sub-partition at <= 168 registers (16 K each)
#define DK_RUNSW_BOUNDS __maxnreg__(168)
#else
#define DK_RUNSW_BOUNDS __launch_bounds__(run_sw_threads<W, D>(), 1)
#endif
__global__ void DK_RUNSW_BOUNDS k_run_sw(const LigDev L, const GridDev g,
                                                                      const ScratchLayout SL, const SearchDev sp,
                                                                      const PopDev pop, const LsArgs a,
                                                                      unsigned long long *prof) {
    namespace cg = cooperative_groups;
    constexpr int NGA = run_sw_threads<W, D>() / W;          // lane groups of the GA phase
    cg::cluster_group cl = cg::this_cluster();
    const int nq = (int)cl.num_blocks(), q = (int)cl.block_rank();
    const int r = blockIdx.x / nq;
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int G = L.G, P = sp.pop;
    const int staged = staged_bytes(L, false);
    const LigSm Ls = stage_ligand(L, sm, staged);
    const int gidx = threadIdx.x / W, sub = threadIdx.x % W;
    uint8_t *gbase = sm + staged + gidx * SL.bytes;
    const Scratch S = scratch_at(gbase, SL);
    const bool timer = prof != nullptr && r == 0 && q == 0 && threadIdx.x == 0;
    // Speculative GA: an offspring slot of the next generation whose four
    // tournament candidates all lie outside this generation's LS sample depends only on data
    // that is final once the GA phase ends (genes / energies of the non-sampled individuals,
    // counter-based words).  CTAs whose Solis-Wets chain has finished score such slots while
    // the run's longer chains still run (they wait at the LS barrier anyway), mark them in the
    // per-parity bitmap, and the next GA phase deals only the rest.  Each slot's arithmetic is
    // that of ga_slot_group whoever computes it, so results are bit-identical.  Scratch: the
    // tree's energy / deviate region (free outside the chain), list capacity kSpecCap slots.
    int *slist = reinterpret_cast<int *>(sm + staged + NGA * SL.bytes);
    constexpr int kSpecCap = 2 * 8 + kTriAhead * kMaxGenes;   // ints of tree_smem's tail (NGA >= 8)
    const bool spec = DK_RUNSW_SPEC && P < kSpecCap && pop.spec_done != nullptr;
    const int SWd = pop.spec_words;
    const uint2 key = make_uint2(sp.key0, sp.key1);
    const uint32_t run_g = (uint32_t)(sp.run_base + r);
    for (;;) {
        RunState st;
        st.evals = __ldcg(&pop.state[r].evals); st.gen = __ldcg(&pop.state[r].gen);
        if (!run_active(st, sp)) break;                   // uniform over the cluster
        // ---- GA phase ----
        const int par = (st.gen + 1) & 1;                 // parity of the generation being created
        if (spec) {
            // the slots still to score: slot 0 (elite + LS pick) and those not marked done
            const unsigned *done = pop.spec_done + ((size_t)r * 2 + par) * SWd;
            if (threadIdx.x < 32) {
                int n = 0;
                for (int w = 0; w < SWd; ++w) {
                    const int k = w * 32 + (int)threadIdx.x;
                    const bool todo = k < P && (k == 0 || !((__ldcg(done + w) >> threadIdx.x) & 1u));
                    const unsigned bal = __ballot_sync(0xffffffffu, todo);
                    if (todo) slist[n + __popc(bal & ((1u << threadIdx.x) - 1u))] = k;
                    n += __popc(bal);
                }
                if (threadIdx.x == 0) slist[kSpecCap - 1] = n;
            }
            __syncthreads();
            const int nrem = slist[kSpecCap - 1];
            for (int base = 0; base < nrem; base += nq * NGA) {
                const int i = base + q * NGA + gidx;
                ga_slot_group<W, MAXC>(Ls, g, S, reinterpret_cast<int *>(gbase + SL.off_extra), sp, pop, G, i < nrem, st,
                                       r, i < nrem ? slist[i] : 0, sub, nullptr);
            }
            if (q == 0 && threadIdx.x == 0) pop.spec_ctr[2 * r + par] = 0;   // this parity's claims are consumed
        } else {
            for (int base = 0; base < P; base += nq * NGA) {
                const int k = base + q * NGA + gidx;
                ga_slot_group<W, MAXC>(Ls, g, S, reinterpret_cast<int *>(gbase + SL.off_extra), sp, pop, G, k < P, st,
                                       r, k < P ? k : 0, sub, nullptr);
            }
        }
        __threadfence();
        cl.sync();
        const unsigned long long t0 = timer ? global_ns() : 0ull;
        // ---- LS phase ----
        if (spec && q == 0)                               // this parity's bitmap is consumed (read above)
            for (int w = threadIdx.x; w < SWd; w += blockDim.x) pop.spec_done[((size_t)r * 2 + par) * SWd + w] = 0u;
        const LsTarget t = ls_target(sp, pop, a, r * nq + q, G);
        sw_tree_chain<W, MAXC, D, 1>(Ls, g, SL, sp, pop, a, t, sm, staged, G);
        if (spec) {
            // next generation g2 = st.gen + 2 (parity par ^ 1): the slots whose candidates avoid
            // this generation's LS sample (pop.perm[r][0, n_ls), written in the GA phase)
            const uint32_t g2 = (uint32_t)st.gen + 2u;
            const int *ls = pop.perm + (size_t)r * P;
            __syncthreads();                              // the chain's reads of the tree region are done
            if (threadIdx.x < 32) {
                int n = 0;
                for (int k0 = 1; k0 < P; k0 += 32) {
                    const int k = k0 + (int)threadIdx.x;
                    bool ok = k < P;
                    if (ok) {
                        const uint4 b0 = stream_block(key, kGA, (uint32_t)k, g2, run_g, 0u);
                        const uint4 b1 = stream_block(key, kGA, (uint32_t)k, g2, run_g, 1u);
                        const uint32_t wv[4] = {b0.x, b0.y, b0.w, b1.x};       // words 0, 1 (A) and 3, 4 (B)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int ci = (int)below(wv[2 * h], (uint32_t)P);
                            int cj = (int)below(wv[2 * h + 1], (uint32_t)(P - 1));
                            if (cj >= ci) cj += 1;
                            for (int s2 = 0; s2 < sp.n_ls; ++s2) {
                                const int m = __ldcg(ls + s2);
                                if (m == ci || m == cj) ok = false;
                            }
                        }
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, ok);
                    if (ok) slist[n + __popc(bal & ((1u << threadIdx.x) - 1u))] = k;
                    n += __popc(bal);
                }
                if (threadIdx.x == 0) slist[kSpecCap - 1] = n;
            }
            __syncthreads();
            const int nspec = slist[kSpecCap - 1];
            RunState st2 = st;
            st2.gen = st.gen + 1;                         // the generation g2 is created from
            int *ctr = pop.spec_ctr + 2 * r + (par ^ 1);
            unsigned *done2 = pop.spec_done + ((size_t)r * 2 + (par ^ 1)) * SWd;
            const int lane = threadIdx.x & 31, wgrp = lane / W;   // lane group within the warp
            for (;;) {
                int c = 0;
                if (lane == 0) c = atomicAdd(ctr, 32 / W);       // one slot per lane group of the warp
                c = __shfl_sync(0xffffffffu, c, 0);
                if (c >= nspec) break;                            // uniform per warp
                const int i = c + wgrp;
                const bool act = i < nspec;
                const int k = act ? slist[i] : 0;
                ga_slot_group<W, MAXC>(Ls, g, S, reinterpret_cast<int *>(gbase + SL.off_extra), sp, pop, G, act, st2,
                                       r, k, sub, nullptr);
                if (act && sub == 0) {
                    __threadfence();
                    atomicOr(done2 + (k >> 5), 1u << (k & 31));
                }
            }
        }
        __threadfence();
        cl.sync();
        if (timer) { prof[0] += global_ns() - t0; prof[1] += 1ull; }
    }
}

#if DK_PART == 1   // non-template kernels: defined in one part only
// ---------------------------------------------------------------------------
// k_gen_end: sum_evals (Listing 1: per-run reduction over the population's
// evaluation counters with warp shuffles) and the generation counter.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gen_end(const SearchDev sp, const PopDev pop) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= sp.runs) return;
    const RunState st = pop.state[r];
    if (!run_active(st, sp)) return;
    long long s = 0;
    for (int i = lane; i < sp.n_ls; i += 32) s += pop.ls_evals[(size_t)r * sp.pop + i];
    s = gsum_ll<32>(s, 0xffffffffu);
    if (lane == 0) {
        pop.state[r].evals = st.evals + (long long)(sp.pop - 1) + s;   // offspring + local search
        pop.state[r].gen = st.gen + 1;
    }
}

// k_best: best of each run's final population (argmin, lowest index on ties).
__global__ void __launch_bounds__(256) k_best(const int G, const SearchDev sp, const PopDev pop, float *bestE,
                                              float *bestG, long long *evals, int *gens) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= sp.runs) return;
    const RunState st = pop.state[r];
    const int buf = st.gen & 1;
    const float *E = pop.E + ((size_t)buf * sp.rstride + r) * sp.pop;
    float bv = INFINITY;
    int bi = 0x7fffffff;
    for (int i = lane; i < sp.pop; i += 32) {
        const float v = nan_inf(E[i]);
        if (v < bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, m);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
        if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const float *row = pop.genes + (((size_t)buf * sp.rstride + r) * sp.pop + bi) * G;
    for (int j = lane; j < G; j += 32) bestG[(size_t)r * G + j] = row[j];
    if (lane == 0) {
        bestE[r] = E[bi];
        if (evals) evals[r] = st.evals;
        if (gens) gens[r] = st.gen;
    }
}

#endif

// ---------------------------------------------------------------------------
// k_bench_part: microbenchmark of one part of the evaluation: PARTS =
// kInter -> pose + grid interpolation (a3+a4, energy + gradient), PARTS = kIntra -> pose
// + pair tiles (a3+a5, energy + forces).  Each group evaluates its genotype `iters`
// times, nudging the translation by 1e-3 Å per iteration (ADADELTA-like locality).
// ---------------------------------------------------------------------------
template <int W, int MAXC, int PARTS, bool PK = false>
__global__ void __launch_bounds__(256, (MAXC <= 4 ? DK_ADA_MINB : 1)) k_bench_part(const LigDev L, const GridDev g,
                                                                                  const ScratchLayout SL, int n, int iters,
                                                                                  const float *__restrict__ genes, float *E) {
    extern __shared__ uint4 smem_u4[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(smem_u4);
    const int gl = threadIdx.x / W, sub = threadIdx.x % W;
    const int gi = blockIdx.x * (blockDim.x / W) + gl;
    const bool act = gi < n;
    if (!__syncthreads_or(act)) return;
    const LigSm Ls = stage_ligand(L, sm, staged_bytes(L, true));
    if (!act) return;
    const Scratch S = scratch_at(sm + staged_bytes(L, true) + gl * SL.bytes, SL);
    const unsigned mask = group_mask<W>();
    for (int j = sub; j < L.G; j += W) S.genes[j] = genes[(size_t)gi * L.G + j];
    __syncwarp(mask);
    float acc = 0.0f;
    for (int it = 0; it < iters; ++it) {
        acc += eval_group<W, MAXC, true, PARTS, 1, PK>(Ls, g, S, sub, mask);
        if (sub == 0) S.genes[0] += 1e-3f;
        __syncwarp(mask);
    }
    if (sub == 0) E[gi] = acc;
}

#if DK_PART == 1
__global__ void k_philox(int n, const uint4 *ctr, const uint2 *key, uint4 *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox4x32_10(ctr[i], key[i]);
}

// k_l2_gather: the L2 gather ceiling of the interpolation kernel: every
// thread issues `iters` rounds of 8 independent random 16-byte loads (__ldg, the corner-
// fetch instruction of inter_atom) over a device-resident buffer of n float4 that fits L2.
// Index: a multiplicative hash of (thread, round, corner).  The checksum keeps the loads live.
__global__ void __launch_bounds__(256) k_l2_gather(const float4 *__restrict__ buf, uint32_t n, int iters,
                                                   float *out) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    uint32_t h = tid * 0x9E3779B9u + 0x7F4A7C15u;
    for (int it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            h = h * 1664525u + 1013904223u;
            v[c] = __ldg(buf + (uint32_t)(((uint64_t)h * n) >> 32));
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) acc += v[c].x + v[c].y + v[c].z + v[c].w;
    }
    if (acc == 1234.5f) out[tid] = acc;
}

__global__ void k_stream_words(uint2 key, uint32_t purpose, uint32_t slot, uint32_t gen, uint32_t run,
                               uint32_t m0, int n, uint32_t *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = stream_word(key, purpose, slot, gen, run, m0 + (uint32_t)i);
}
#endif

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
#define DK_DISPATCH(cfg, ...)                                                \
    do {                                                                     \
        if ((cfg).W == 16) { constexpr int W = 16, MAXC = 1; __VA_ARGS__; }  \
        else switch ((cfg).MAXC) {                                           \
            case 1: { constexpr int W = 32, MAXC = 1; __VA_ARGS__; } break;  \
            case 2: { constexpr int W = 32, MAXC = 2; __VA_ARGS__; } break;  \
            case 3: { constexpr int W = 32, MAXC = 3; __VA_ARGS__; } break;  \
            case 4: { constexpr int W = 32, MAXC = 4; __VA_ARGS__; } break;  \
            default: { constexpr int W = 32, MAXC = 8; __VA_ARGS__; } break; \
        }                                                                    \
    } while (0)

// The packed FP32x2 gradient tiles (score.cuh, LigDev::packed: D5, W = 32, two chunks:
// 49 <= N <= 64 with the second one padded, 65 <= N <= ~82 with a hybrid tail) are a
// compile-time variant (PK) of the gradient kernels: DK_IF_PACKED(L, cfg, body) runs body
// with W = 32, MAXC = 2 or 3, PK = true for a packed ligand, else falls through to the
// statement that follows it.
#ifdef DK_PACK_ON
#define DK_IF_PACKED(L, cfg, ...)                                                              \
    if ((L).packed && (cfg).W == 32 && (cfg).MAXC == 3) {                                      \
        constexpr int W = 32, MAXC = 3;                                                        \
        constexpr bool PK = true;                                                              \
        __VA_ARGS__;                                                                           \
    } else if ((L).packed && (cfg).W == 32 && (cfg).MAXC == 2) {                               \
        constexpr int W = 32, MAXC = 2;                                                        \
        constexpr bool PK = true;                                                              \
        __VA_ARGS__;                                                                           \
    } else
#else
#define DK_IF_PACKED(L, cfg, ...)
#endif

static constexpr int kThreads = 256;
static constexpr int kSmemMax = 227 * 1024;

template <typename K>
static cudaError_t allow_smem(K kernel) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
}

#if DK_PART == 3 || DK_PART == 4
// cooperative SW trees exist for 32-lane groups only
template <int W, int MAXC, bool TRACE>
static cudaError_t allow_split() {
    if constexpr (W == 32) {
        cudaError_t e = allow_smem(k_ls_sw_tree<W, MAXC, 1, 4, TRACE>);
        return e == cudaSuccess ? allow_smem(k_ls_sw_tree<W, MAXC, 2, 2, TRACE>) : e;
    }
    return cudaSuccess;
}

template <int W, int MAXC, bool TRACE>
static cudaError_t allow_sw() {
    cudaError_t e = allow_smem(k_ls_sw<W, MAXC, TRACE>);
    if (e == cudaSuccess) e = allow_smem(k_ls_sw_tree<W, MAXC, 2, 1, TRACE>);
    if (e == cudaSuccess) e = allow_smem(k_ls_sw_tree<W, MAXC, 3, 1, TRACE>);
    if (e == cudaSuccess) e = allow_split<W, MAXC, TRACE>();
    return e;
}

#endif

static inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

#if DK_PART == 1
cudaError_t launch_ls(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, const LsArgs &a,
                      int n_total, cudaStream_t s) {
    if (n_total <= 0) return cudaSuccess;
    return sp.ls_method == 1 ? launch_ls_sw(L, g, sp, pop, a, n_total, s)
                             : launch_ls_adadelta(L, g, sp, pop, a, n_total, s);
}

cudaError_t setup_kernel_attributes() {
    cudaError_t e = cudaSuccess;
#define DK_ATTR(W, MAXC)                                                             \
    if (e == cudaSuccess) e = allow_smem(k_eval<W, MAXC, false>);                    \
    if (e == cudaSuccess) e = allow_smem(k_eval<W, MAXC, true>);                     \
    if (e == cudaSuccess) e = allow_smem(k_eval<W, MAXC, false, kInter>);            \
    if (e == cudaSuccess) e = allow_smem(k_eval<W, MAXC, false, kIntra>);            \
    if (e == cudaSuccess) e = allow_smem(k_init<W, MAXC>);                           \
    if (e == cudaSuccess) e = allow_smem(k_ga<W, MAXC>);                             \
    if (e == cudaSuccess) e = allow_smem(k_bench_part<W, MAXC, kInter>);             \
    if (e == cudaSuccess) e = allow_smem(k_bench_part<W, MAXC, kIntra>);
    DK_ATTR(16, 1) DK_ATTR(32, 1) DK_ATTR(32, 2) DK_ATTR(32, 3) DK_ATTR(32, 4) DK_ATTR(32, 8)
#undef DK_ATTR
#ifdef DK_PACK_ON
    if (e == cudaSuccess) e = allow_smem(k_eval<32, 3, true, kAll, true>);
    if (e == cudaSuccess) e = allow_smem(k_bench_part<32, 3, kIntra, true>);
    if (e == cudaSuccess) e = allow_smem(k_eval<32, 2, true, kAll, true>);
    if (e == cudaSuccess) e = allow_smem(k_bench_part<32, 2, kIntra, true>);
#endif
    if (e == cudaSuccess) e = setup_attributes_adadelta();
    if (e == cudaSuccess) e = setup_attributes_sw();
    return e;
}
#endif

#if DK_PART == 2
cudaError_t setup_attributes_adadelta() {
    cudaError_t e = cudaSuccess;
#define DK_ATTR(W, MAXC)                                                             \
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<W, MAXC>);                    \
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<W, MAXC, true>);
    DK_ATTR(16, 1) DK_ATTR(32, 1) DK_ATTR(32, 2) DK_ATTR(32, 3) DK_ATTR(32, 4) DK_ATTR(32, 8)
#undef DK_ATTR
#ifdef DK_PACK_ON
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<32, 3, false, true>);
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<32, 3, true, true>);
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<32, 2, false, true>);
    if (e == cudaSuccess) e = allow_smem(k_ls_adadelta<32, 2, true, true>);
#endif
    return e;
}
#endif

#if DK_PART == 3
cudaError_t setup_attributes_sw() {
    cudaError_t e = cudaSuccess;
#define DK_ATTR(W, MAXC)                                                             \
    if (e == cudaSuccess) e = allow_sw<W, MAXC, false>();                            \
    if (e == cudaSuccess) e = allow_smem(k_run_sw<W, MAXC, 2>);                      \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_run_sw<W, MAXC, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
    if (e == cudaSuccess) e = allow_smem(k_run_sw<W, MAXC, 3>);                      \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_run_sw<W, MAXC, 3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    DK_ATTR(16, 1) DK_ATTR(32, 1) DK_ATTR(32, 2) DK_ATTR(32, 3) DK_ATTR(32, 4) DK_ATTR(32, 8)
#undef DK_ATTR
    return e == cudaSuccess ? setup_attributes_sw_trace() : e;
}
#endif

#if DK_PART == 4
cudaError_t setup_attributes_sw_trace() {
    cudaError_t e = cudaSuccess;
#define DK_ATTR(W, MAXC) if (e == cudaSuccess) e = allow_sw<W, MAXC, true>();
    DK_ATTR(16, 1) DK_ATTR(32, 1) DK_ATTR(32, 2) DK_ATTR(32, 3) DK_ATTR(32, 4) DK_ATTR(32, 8)
#undef DK_ATTR
    return e;
}
#endif

#if DK_PART == 1
cudaError_t launch_eval(const LigDev &L, const GridDev &g, int n, const float *genes, float *E, float *grad,
                        float *xyz, const int *dfs2orig, cudaStream_t s, int parts) {
    if (n <= 0) return cudaSuccess;
    const GroupCfg cfg = pick_group(L.N);
    const bool want_grad = grad != nullptr;
    const ScratchLayout SL = scratch_layout(L, want_grad, 0);
    const int groups = kThreads / cfg.W;
    const size_t smem = (size_t)staged_bytes(L, want_grad) + (size_t)groups * SL.bytes;
    if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
    const int blocks = ceil_div(n, groups);
    DK_DISPATCH(cfg, {
        // parts = one term only (dock_eval_terms): energy-only kernels of that term
        if (parts == kInter && !want_grad)
            k_eval<W, MAXC, false, kInter><<<blocks, kThreads, smem, s>>>(L, g, SL, n, genes, E, nullptr, xyz, dfs2orig);
        else if (parts == kIntra && !want_grad)
            k_eval<W, MAXC, false, kIntra><<<blocks, kThreads, smem, s>>>(L, g, SL, n, genes, E, nullptr, xyz, dfs2orig);
        else if (want_grad) {
            DK_IF_PACKED(L, cfg, { k_eval<W, MAXC, true, kAll, PK><<<blocks, kThreads, smem, s>>>(L, g, SL, n, genes, E, grad, xyz, dfs2orig); })
            k_eval<W, MAXC, true><<<blocks, kThreads, smem, s>>>(L, g, SL, n, genes, E, grad, xyz, dfs2orig);
        }
        else k_eval<W, MAXC, false><<<blocks, kThreads, smem, s>>>(L, g, SL, n, genes, E, grad, xyz, dfs2orig);
    });
    return cudaGetLastError();
}

cudaError_t launch_init(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, cudaStream_t s) {
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, false, 0);
    const int groups = kThreads / cfg.W;
    const size_t smem = (size_t)staged_bytes(L, false) + (size_t)groups * SL.bytes;
    if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
    const int blocks = ceil_div((long long)sp.runs * sp.pop, groups);
    DK_DISPATCH(cfg, { k_init<W, MAXC><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop); });
    return cudaGetLastError();
}

cudaError_t launch_ga(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, int *dbg,
                      cudaStream_t s) {
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, false, 4 * sp.pop);
    const int groups = kThreads / cfg.W;
    const size_t smem = (size_t)staged_bytes(L, false) + (size_t)groups * SL.bytes;
    if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
    const int blocks = ceil_div((long long)sp.runs * sp.pop, groups);
    DK_DISPATCH(cfg, { k_ga<W, MAXC><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop, dbg); });
    return cudaGetLastError();
}

#endif

#if DK_PART == 3 || DK_PART == 4
// shared memory of a k_ls_sw_tree<.., D, KP> CTA: ligand block, one scratch per lane
// group, x and b, the partial energies and the double-buffered deviate shapes
static size_t tree_smem(const LigDev &L, const ScratchLayout &SL, int D, int KP) {
    const int ngr = (D == 3 ? 26 : (D == 2 ? 8 : 2)) * KP;
    return (size_t)staged_bytes(L, false) + (size_t)ngr * SL.bytes + 4 * (2 * ngr + kTriAhead * kMaxGenes);
}

// k_run_sw: the tree's shared memory, or the GA phase's scratch of all its lane groups
static size_t run_sw_smem(const LigDev &L, const ScratchLayout &SL, int D) {
    const int nga = (D == 3 ? run_sw_threads<16, 3>() : run_sw_threads<16, 2>()) / 16;   // W = 16: most groups
    const size_t ga = (size_t)staged_bytes(L, false) + (size_t)nga * SL.bytes;
    const size_t tr = tree_smem(L, SL, D, 1);
    return ga > tr ? ga : tr;
}

// TR = true: the parity-hook (TRACE) instantiations, compiled in part 4.
#define DK_TRACE_SEL(...)                                                          \
    do { __VA_ARGS__; } while (0)

template <bool TR>
cudaError_t launch_ls_sw_t(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, const LsArgs &a,
                           int n_total, cudaStream_t s) {
    const GroupCfg cfg = pick_group(L.N);
    {
        const ScratchLayout SL = scratch_layout(L, false, 0);
        // (A full warp per node for W = 16 ligands -- half the pairs per lane -- was measured
        // 0.63x on 1stp: twice the warps per round, same critical path.)
        const GroupCfg tcfg = cfg;
        // Speculation depth: the deepest tree whose CTAs are all co-resident (one wave);
        // a full launch gains nothing from speculation and uses the plain kernel.
        int depth = sp.sw_depth;
        if (depth == 0) {
            depth = 1;
            int dev = 0, nsm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            // Measured on B200 (profiles/r01n, NEXT-1 sweep): depth 2 wins whenever its CTAs
            // fit one wave (1stp 1.7x, PS/PM/PL with 10 runs 2.0x / 2.4x / 3.6x) and, for
            // large ligands (P >= 2000, PL), up to ~4 waves (1.43x at 900 chains); small
            // ligands at 900 chains prefer depth 1 (0.91x / 0.96x).  Depth 3 (26 groups)
            // never won (issue contention, spills at the 2-CTA/SM register cap).
            for (int D = 2; D >= 2 && depth == 1; --D) {
                const int ngr = D == 3 ? 26 : 8;
                const size_t sm_b = tree_smem(L, SL, D, 1);
                int per_sm = 0;
                DK_DISPATCH(tcfg, {
                    if (D == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ls_sw_tree<W, MAXC, 3>, tree_threads<W, 3>(), sm_b);
                    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ls_sw_tree<W, MAXC, 2>, tree_threads<W, 2>(), sm_b);
                });
                cudaGetLastError();
                const long long waves = L.P >= 2000 ? 4 : 1;
                const long long in_flight = a.wave_total > 0 ? a.wave_total : n_total;
                if (sm_b <= (size_t)kSmemMax && per_sm > 0 && in_flight <= waves * per_sm * nsm) depth = D;
            }
        }
        // Cooperative evaluation (several warps per trial point) for large ligands, whose one
        // evaluation is the chain latency: split 2 with depth 2, or split 4 with depth 1.
        // Measured (profiles/next1): PL (P = 5,358) 4 warps x depth 1 beats depth 2 by 1.27x
        // (10 runs) and 1.24x (100 runs); PM (P ~ 700) is best without splitting.
        int split = sp.sw_split;
        if (split == 0) split = (L.P >= 2000 && sp.sw_depth == 0) ? 4 : 1;
        if (tcfg.W != 32 || (split != 2 && split != 4)) split = 1;
        if (split > 1) {
            const int D = split == 2 ? 2 : 1;
            const size_t smem = tree_smem(L, SL, D, split);
            if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
            switch (tcfg.MAXC) {
#define DK_SPLIT(M)                                                                                     \
    case M:                                                                                             \
        DK_TRACE_SEL(if (split == 2) k_ls_sw_tree<32, M, 2, 2, TR><<<n_total, tree_threads<32, 2, 2>(), smem, s>>>(L, g, SL, sp, pop, a); \
                     else k_ls_sw_tree<32, M, 1, 4, TR><<<n_total, tree_threads<32, 1, 4>(), smem, s>>>(L, g, SL, sp, pop, a)); \
        break;
                DK_SPLIT(1) DK_SPLIT(2) DK_SPLIT(3) DK_SPLIT(4)
                default: DK_SPLIT(8)
#undef DK_SPLIT
            }
            return cudaGetLastError();
        }
        if (depth >= 2) {
            const size_t smem = tree_smem(L, SL, depth, 1);
            if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
            DK_DISPATCH(tcfg, { DK_TRACE_SEL(
                if (depth == 3) k_ls_sw_tree<W, MAXC, 3, 1, TR><<<n_total, tree_threads<W, 3>(), smem, s>>>(L, g, SL, sp, pop, a);
                else k_ls_sw_tree<W, MAXC, 2, 1, TR><<<n_total, tree_threads<W, 2>(), smem, s>>>(L, g, SL, sp, pop, a)); });
            return cudaGetLastError();
        }
        // depth 1: one warp per individual; few individuals -> one warp per CTA so they
        // spread over all SMs.
        const int ng = cfg.W <= 16 ? 2 : 1;
        const int warps = (a.wave_total > 0 ? a.wave_total : n_total) >= 148 * 8 ? 8 : 1;
        const size_t smem = (size_t)staged_bytes(L, false) + (size_t)warps * ng * SL.bytes;
        if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
        const int blocks = ceil_div(n_total, warps);
        DK_DISPATCH(cfg, { DK_TRACE_SEL(k_ls_sw<W, MAXC, TR><<<blocks, warps * 32, smem, s>>>(L, g, SL, sp, pop, a)); });
    }
    return cudaGetLastError();
}
#if DK_PART == 4
template cudaError_t launch_ls_sw_t<true>(const LigDev &, const GridDev &, const SearchDev &, const PopDev &,
                                         const LsArgs &, int, cudaStream_t);
#else
cudaError_t launch_ls_sw(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop, const LsArgs &a,
                         int n_total, cudaStream_t s) {
    return a.sw_trace ? launch_ls_sw_t<true>(L, g, sp, pop, a, n_total, s)
                      : launch_ls_sw_t<false>(L, g, sp, pop, a, n_total, s);
}

// Persistent cluster engine (k_run_sw): eligible when the run's LS individuals fit one
// cluster (n_ls <= 16), no cooperative split is wanted, and the speculation-depth rule
// would pick depth 2 for all runs' chains (so the results and the tree are those of the
// lockstep engine).  Returns 0 if not eligible.
int run_sw_eligible(const LigDev &L, const SearchDev &sp) {
    if (sp.ls_method != 1 || sp.n_ls < 1 || sp.n_ls > 16 || sp.ls_iters < 1) return 0;
    if (sp.sw_depth != 0 && sp.sw_depth != 2 && sp.sw_depth != 3) return 0;
    if (sp.sw_split == 2 || sp.sw_split == 4 || (sp.sw_split == 0 && L.P >= 2000 && pick_group(L.N).W == 32)) return 0;
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, false, 4 * sp.pop);
    const size_t smem = run_sw_smem(L, SL, sp.sw_depth == 3 ? 3 : 2);
    if (smem > (size_t)kSmemMax) return 0;
#ifndef DK_RUNSW_ANY
#define DK_RUNSW_ANY 0   // experiment build only (scripts/variants.py): lift the one-wave condition
#endif
    if (sp.sw_depth == 0 && !DK_RUNSW_ANY) {   // the auto depth rule of launch_ls, on all runs' chains
        int dev = 0, nsm = 148, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const size_t sm_b = tree_smem(L, scratch_layout(L, false, 0), 2, 1);
        DK_DISPATCH(cfg, { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ls_sw_tree<W, MAXC, 2>, tree_threads<W, 2>(), sm_b); });
        cudaGetLastError();
        const long long waves = L.P >= 2000 ? 4 : 1;
        if (!(per_sm > 0 && (long long)sp.runs * sp.n_ls <= waves * per_sm * nsm)) return 0;
    }
    // the cluster shape must be schedulable at all (n_ls CTAs of this size in one GPC)
    int clusters = 0;
    DK_DISPATCH(cfg, {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)sp.n_ls);
        const bool d3 = sp.sw_depth == 3;
        lc.blockDim = dim3(d3 ? run_sw_threads<W, 3>() : run_sw_threads<W, 2>());
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)sp.n_ls; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.attrs = at; lc.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&clusters, d3 ? k_run_sw<W, MAXC, 3> : k_run_sw<W, MAXC, 2>, &lc) !=
            cudaSuccess)
            clusters = 0;
    });
    cudaGetLastError();
    return clusters > 0 ? 1 : 0;
}

cudaError_t launch_run_sw(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                          unsigned long long *prof, cudaStream_t s) {
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, false, 4 * sp.pop);
    const int D = sp.sw_depth == 3 ? 3 : 2;   // depth 3 only on request (sw_depth = 3)
    const size_t smem = run_sw_smem(L, SL, D);
    LsArgs a{};
    a.use_state = 1; a.n_per_run = sp.n_ls; a.iters = sp.ls_iters;
    cudaError_t e = cudaSuccess;
    DK_DISPATCH(cfg, {
        auto kern = D == 3 ? k_run_sw<W, MAXC, 3> : k_run_sw<W, MAXC, 2>;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(sp.runs * sp.n_ls));
        lc.blockDim = dim3(D == 3 ? run_sw_threads<W, 3>() : run_sw_threads<W, 2>());
        lc.dynamicSmemBytes = smem;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)sp.n_ls; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.attrs = at; lc.numAttrs = 1;
        e = cudaLaunchKernelEx(&lc, kern, L, g, SL, sp, pop, a, prof);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}
#endif  // DK_PART == 3 (launch_ls_sw .. launch_run_sw)
#endif  // DK_PART == 3 || DK_PART == 4

#if DK_PART == 2
// Lane groups of k_ls_adadelta resident on the whole device (occupancy x SMs x groups per
// CTA): the engine's auto rule compares one generation's LS individuals with it.
int adadelta_resident_groups(const LigDev &L) {
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, true, 0);
    const int groups = kThreads / cfg.W;
    const size_t smem = (size_t)staged_bytes(L, true) + (size_t)groups * SL.bytes;
    int dev = 0, nsm = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    DK_IF_PACKED(L, cfg, { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ls_adadelta<W, MAXC, false, PK>, kThreads, smem); })
    DK_DISPATCH(cfg, { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ls_adadelta<W, MAXC>, kThreads, smem); });
    cudaGetLastError();
    return per_sm * nsm * groups;
}

cudaError_t launch_ls_adadelta(const LigDev &L, const GridDev &g, const SearchDev &sp, const PopDev &pop,
                               const LsArgs &a, int n_total, cudaStream_t s) {
    const GroupCfg cfg = pick_group(L.N);
    {
        const ScratchLayout SL = scratch_layout(L, true, 0);
        const int groups = kThreads / cfg.W;
        const size_t smem = (size_t)staged_bytes(L, true) + (size_t)groups * SL.bytes;
        if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
        const int blocks = ceil_div(n_total, groups);
        if (a.ad_trace_x) {
            DK_IF_PACKED(L, cfg, { k_ls_adadelta<W, MAXC, true, PK><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop, a); })
            DK_DISPATCH(cfg, { k_ls_adadelta<W, MAXC, true><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop, a); });
        } else {
            DK_IF_PACKED(L, cfg, { k_ls_adadelta<W, MAXC, false, PK><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop, a); })
            DK_DISPATCH(cfg, { k_ls_adadelta<W, MAXC><<<blocks, kThreads, smem, s>>>(L, g, SL, sp, pop, a); });
        }
    }
    return cudaGetLastError();
}

#endif

#if DK_PART == 1
cudaError_t launch_bench_part(const LigDev &L, const GridDev &g, int part, int n, int iters, const float *genes,
                              float *E, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const GroupCfg cfg = pick_group(L.N);
    const ScratchLayout SL = scratch_layout(L, true, 0);
    const int groups = kThreads / cfg.W;
    const size_t smem = (size_t)staged_bytes(L, true) + (size_t)groups * SL.bytes;
    if (smem > (size_t)kSmemMax) return cudaErrorInvalidConfiguration;
    const int blocks = ceil_div(n, groups);
    DK_IF_PACKED(L, cfg, {
        if (part == 0) k_bench_part<W, MAXC, kInter><<<blocks, kThreads, smem, s>>>(L, g, SL, n, iters, genes, E);
        else k_bench_part<W, MAXC, kIntra, PK><<<blocks, kThreads, smem, s>>>(L, g, SL, n, iters, genes, E);
    })
    DK_DISPATCH(cfg, {
        if (part == 0) k_bench_part<W, MAXC, kInter><<<blocks, kThreads, smem, s>>>(L, g, SL, n, iters, genes, E);
        else k_bench_part<W, MAXC, kIntra><<<blocks, kThreads, smem, s>>>(L, g, SL, n, iters, genes, E);
    });
    return cudaGetLastError();
}

cudaError_t launch_gen_end(const SearchDev &sp, const PopDev &pop, cudaStream_t s) {
    k_gen_end<<<ceil_div(sp.runs, kThreads / 32), kThreads, 0, s>>>(sp, pop);
    return cudaGetLastError();
}

cudaError_t launch_best(const LigDev &L, const SearchDev &sp, const PopDev &pop, float *bestE, float *bestG,
                        long long *evals, int *gens, cudaStream_t s) {
    k_best<<<ceil_div(sp.runs, kThreads / 32), kThreads, 0, s>>>(L.G, sp, pop, bestE, bestG, evals, gens);
    return cudaGetLastError();
}

cudaError_t launch_philox(int n, const uint32_t *ctr, const uint32_t *key, uint32_t *out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_philox<<<ceil_div(n, 128), 128, 0, s>>>(n, reinterpret_cast<const uint4 *>(ctr),
                                              reinterpret_cast<const uint2 *>(key), reinterpret_cast<uint4 *>(out));
    return cudaGetLastError();
}

cudaError_t launch_l2_gather(const float4 *buf, uint32_t n, int blocks, int iters, float *out, cudaStream_t s) {
    k_l2_gather<<<blocks, 256, 0, s>>>(buf, n, iters, out);
    return cudaGetLastError();
}

cudaError_t launch_stream_words(uint32_t k0, uint32_t k1, uint32_t purpose, uint32_t slot, uint32_t gen, uint32_t run,
                                uint32_t m0, int n, uint32_t *out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_stream_words<<<ceil_div(n, 128), 128, 0, s>>>(make_uint2(k0, k1), purpose, slot, gen, run, m0, n, out);
    return cudaGetLastError();
}

#endif

}  // namespace DK_SF_NS
}  // namespace dk
