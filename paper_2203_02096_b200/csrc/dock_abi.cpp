// dock_abi.cpp — the C ABI (include/dock.h) and the per-device engine.
//
// The engine keeps the whole search on the device: populations, per-run counters and the
// LS sample live in HBM; one generation = k_ga -> k_ls_* -> k_gen_end, captured as a
// CUDA graph of `gens_per_graph` generations and relaunched until every run has met its
// evaluation budget (D8.5).  The host reads 16 bytes per run per graph launch to
// decide termination; finished runs turn their kernels into no-ops.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cluster.cuh"
#include "engine.h"

namespace {

thread_local std::string g_init_error;

// DOCK_TRACE=1: wall time of host-side phases to stderr (diagnostics of the e2e path).
struct Trace {
    const char *name;
    std::chrono::steady_clock::time_point t0;
    static bool on() {
        static const bool v = std::getenv("DOCK_TRACE") != nullptr;
        return v;
    }
    explicit Trace(const char *n) : name(n), t0(std::chrono::steady_clock::now()) {}
    ~Trace() {
        if (on())
            std::fprintf(stderr, "[dock] %s %.3f ms\n", name,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            c->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
            return DOCK_E_INTERNAL;                                                       \
        }                                                                                 \
    } while (0)

int input_error(dock_ctx *c, const std::string &m) {
    if (c) c->err = m;
    return DOCK_E_INPUT;
}

// n_ls = ceil(ls_rate * pop - 1e-4) clamped to [0, pop] (DESIGN.md §3 reading 16a).
int n_ls_of(float ls_rate, int pop) {
    int n = (int)std::ceil((double)ls_rate * (double)pop - 1e-4);
    return std::max(0, std::min(pop, n));
}

dk::SearchDev make_search(const dock_ctx *c, int pop, int runs, int run_base, uint32_t ligand_id, int64_t max_evals,
                          uint64_t seed) {
    const dock_params &p = c->params;
    dk::SearchDev s{};
    s.p_tour = p.p_tour; s.p_cross = p.p_cross; s.p_mut = p.p_mut;
    s.mut_trans = p.mut_trans; s.mut_angle = p.mut_angle;
    s.ls_method = p.ls_method; s.ls_iters = p.ls_max_iters; s.n_ls = n_ls_of(p.ls_rate, pop);
    s.sw_rho = p.sw_rho; s.sw_rho_min = p.sw_rho_min; s.sw_expand = p.sw_expand; s.sw_contract = p.sw_contract;
    s.sw_cons_succ = p.sw_cons_succ; s.sw_cons_fail = p.sw_cons_fail;
    s.sw_depth = p.sw_depth;
    s.sw_split = p.sw_split;
    s.ad_rho = p.ad_rho; s.ad_eps = p.ad_eps;
    s.max_generations = p.max_generations;
    s.max_evals = max_evals;
    s.pop = pop; s.runs = runs; s.run_base = run_base; s.rstride = runs;
    const uint64_t k = seed + (uint64_t)ligand_id * 0x9E3779B97F4A7C15ull;   // D2 key
    s.key0 = (uint32_t)k; s.key1 = (uint32_t)(k >> 32);
    return s;
}

dk::PopDev pop_of(const dock_ctx *c) {
    dk::PopDev d;
    d.genes = c->d_genes; d.E = c->d_E; d.state = c->d_state; d.perm = c->d_perm; d.ls_evals = c->d_ls_evals;
    d.ls_count = c->d_ls_count;
    d.spec_done = c->d_spec_done; d.spec_ctr = c->d_spec_ctr; d.spec_words = (c->cap_pop + 31) / 32;
    return d;
}

int ensure_buffers(dock_ctx *c, int runs, int pop) {
    if (runs <= c->cap_runs && pop <= c->cap_pop) return DOCK_OK;
    const int R = std::max(runs, c->cap_runs), P = std::max(pop, c->cap_pop);
    CK(dk::after_last_use(c, c->stream));   // kernels of an earlier asynchronous call may still use them
    CK(cudaStreamSynchronize(c->stream));
    dk::dfree(c->d_genes, c->stream); dk::dfree(c->d_E, c->stream); dk::dfree(c->d_state, c->stream);
    dk::dfree(c->d_perm, c->stream); dk::dfree(c->d_ls_evals, c->stream); dk::dfree(c->d_ls_count, c->stream);
    dk::dfree(c->d_spec_done, c->stream); dk::dfree(c->d_spec_ctr, c->stream);
    c->d_genes = nullptr; c->d_E = nullptr; c->d_state = nullptr; c->d_perm = nullptr; c->d_ls_evals = nullptr;
    c->d_ls_count = nullptr; c->d_spec_done = nullptr; c->d_spec_ctr = nullptr;
    c->cap_runs = c->cap_pop = 0;
    // rows are strided by the ligand's G, but sized for the largest G so a context can be
    // reused for any ligand (dock_screen slots)
    const size_t G = (size_t)dk::kMaxGenes;
    cudaStream_t s = c->stream;
    CK(dk::dmalloc((void **)&c->d_genes, 2 * (size_t)R * P * G * sizeof(float), s));
    CK(dk::dmalloc((void **)&c->d_E, 2 * (size_t)R * P * sizeof(float), s));
    CK(dk::dmalloc((void **)&c->d_state, (size_t)R * sizeof(dk::RunState), s));
    CK(dk::dmalloc((void **)&c->d_perm, (size_t)R * P * sizeof(int), s));
    CK(dk::dmalloc((void **)&c->d_ls_evals, (size_t)R * P * sizeof(int), s));
    CK(dk::dmalloc((void **)&c->d_ls_count, (size_t)R * sizeof(int), s));
    CK(cudaMemsetAsync(c->d_ls_count, 0, (size_t)R * sizeof(int), s));
    const size_t spw = (size_t)(P + 31) / 32;
    CK(dk::dmalloc((void **)&c->d_spec_done, (size_t)R * 2 * spw * sizeof(unsigned), s));
    CK(dk::dmalloc((void **)&c->d_spec_ctr, (size_t)R * 2 * sizeof(int), s));
    CK(cudaStreamSynchronize(s));   // usable from any stream (dock_run_device's) from here on
    if (!c->h_state.reserve(R)) { c->err = "pinned host allocation failed"; return DOCK_E_INTERNAL; }
    c->cap_runs = R; c->cap_pop = P;
    return DOCK_OK;
}

int check_run_args(dock_ctx *c, int pop, int runs, int run_base, int64_t max_evals) {
    if (pop < 2 || pop > 4096) return input_error(c, "pop_size: must be in 2..4096");
    if (runs < 1) return input_error(c, "num_runs: must be >= 1");
    if (run_base < 0) return input_error(c, "run_base: must be >= 0");
    if (max_evals < pop) return input_error(c, "max_evals: must be >= pop_size");
    return DOCK_OK;
}

// Scratch buffer of a hook call: pool-allocated on the call's stream, freed on it (the
// hooks synchronise that stream before returning).
struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    explicit DevBuf(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t bytes) { return dk::dmalloc(&p, bytes, s); }
    ~DevBuf() { dk::dfree(p, s); }
};

}  // namespace

namespace dk {

bool prob_ok(float p) { return std::isfinite(p) && p >= 0.f && p <= 1.f; }

cudaError_t after_last_use(dock_ctx *c, cudaStream_t s) {
    return c->last_use ? cudaStreamWaitEvent(s, c->last_use, 0) : cudaSuccess;
}

cudaError_t mark_last_use(dock_ctx *c, cudaStream_t s) {
    return c->last_use ? cudaEventRecord(c->last_use, s) : cudaSuccess;
}

int validate_params(const dock_params &p, std::string *err) {
    if (!prob_ok(p.p_tour) || !prob_ok(p.p_cross) || !prob_ok(p.p_mut)) { *err = "params: probabilities must be in [0,1]"; return DOCK_E_INPUT; }
    if (!std::isfinite(p.mut_trans) || !std::isfinite(p.mut_angle) || p.mut_trans < 0 || p.mut_angle < 0) { *err = "params.mut_*: must be finite, >= 0"; return DOCK_E_INPUT; }
    if (p.ls_method != DOCK_LS_ADADELTA && p.ls_method != DOCK_LS_SOLIS_WETS) { *err = "params.ls_method: 0 or 1"; return DOCK_E_INPUT; }
    if (!prob_ok(p.ls_rate)) { *err = "params.ls_rate: must be in [0,1]"; return DOCK_E_INPUT; }
    if (p.ls_max_iters < 0) { *err = "params.ls_max_iters: must be >= 0"; return DOCK_E_INPUT; }
    if (!(p.sw_rho > 0) || !(p.sw_rho_min > 0) || !(p.sw_expand > 0) || !(p.sw_contract > 0) || p.sw_cons_succ < 1 || p.sw_cons_fail < 1) { *err = "params.sw_*: must be positive"; return DOCK_E_INPUT; }
    if (!(p.ad_rho >= 0 && p.ad_rho < 1) || !(p.ad_eps > 0)) { *err = "params.ad_rho in [0,1), ad_eps > 0"; return DOCK_E_INPUT; }
    if (p.max_generations < 0) { *err = "params.max_generations: must be >= 0"; return DOCK_E_INPUT; }
    if (p.gens_per_graph < 1 || p.gens_per_graph > 4096) { *err = "params.gens_per_graph: 1..4096"; return DOCK_E_INPUT; }
    if (p.sw_depth < 0 || p.sw_depth > 3) { *err = "params.sw_depth: 0..3"; return DOCK_E_INPUT; }
    if (p.sw_split != 0 && p.sw_split != 1 && p.sw_split != 2 && p.sw_split != 4) { *err = "params.sw_split: 0, 1, 2 or 4"; return DOCK_E_INPUT; }
    if (p.run_branches < 0 || p.run_branches > 3) { *err = "params.run_branches: 0..3"; return DOCK_E_INPUT; }
    if (p.scoring != DOCK_SF_D5 && p.scoring != DOCK_SF_AD4) { *err = "params.scoring: DOCK_SF_D5 or DOCK_SF_AD4"; return DOCK_E_INPUT; }
    for (float w : {p.w_vdw, p.w_hb, p.w_el, p.w_ds, p.w_tors, p.qasp})
        if (!std::isfinite(w) || w < 0.f) { *err = "params.w_* / qasp: must be finite and >= 0"; return DOCK_E_INPUT; }
    return DOCK_OK;
}

namespace {
std::mutex g_pinned_mu;
std::vector<std::pair<size_t, void *>> g_pinned_free;   // (size class, block)
size_t pinned_class(size_t b) {
    size_t c = 256;
    while (c < b) c <<= 1;
    return c;
}
}  // namespace

void *pinned_get(size_t bytes) {
    const size_t cls = pinned_class(bytes);
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        for (size_t i = 0; i < g_pinned_free.size(); ++i)
            if (g_pinned_free[i].first == cls) {
                void *p = g_pinned_free[i].second;
                g_pinned_free.erase(g_pinned_free.begin() + i);
                return p;
            }
    }
    void *p = nullptr;
    if (cudaMallocHost(&p, cls) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return p;
}

void pinned_put(void *p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back({pinned_class(bytes), p});
}

void pool_setup(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    done.push_back(device);
}

Receptor::~Receptor() {
    cudaSetDevice(device);
    dfree(d_maps, stream);
    if (stream) cudaStreamDestroy(stream);
}

int receptor_upload(const dock_grids *grids, const std::vector<float4> &packed, int device,
                    std::shared_ptr<Receptor> *out, std::string *err) {
    auto r = std::make_shared<Receptor>();
    r->device = device;
    r->bytes = packed.size() * sizeof(float4);
    if (cudaSetDevice(device) != cudaSuccess ||
        (pool_setup(device), cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        dmalloc((void **)&r->d_maps, r->bytes, r->stream) != cudaSuccess ||
        cudaMemcpyAsync(r->d_maps, packed.data(), r->bytes, cudaMemcpyHostToDevice, r->stream) != cudaSuccess ||
        cudaStreamSynchronize(r->stream) != cudaSuccess) {
        cudaGetLastError();
        *err = "receptor upload to device " + std::to_string(device) + " failed";
        return DOCK_E_INTERNAL;
    }
    GridDev &g = r->grid;
    g.maps = r->d_maps;
    g.nx = grids->nx; g.ny = grids->ny; g.nz = grids->nz; g.n_types = grids->n_types;
    g.ox = grids->origin[0]; g.oy = grids->origin[1]; g.oz = grids->origin[2];
    g.s = grids->spacing; g.inv_s = 1.0f / grids->spacing;
    g.hx = g.ox + (float)(g.nx - 1) * g.s; g.hy = g.oy + (float)(g.ny - 1) * g.s; g.hz = g.oz + (float)(g.nz - 1) * g.s;
    *out = std::move(r);
    return DOCK_OK;
}

int ctx_create(std::shared_ptr<Receptor> rec, const dock_params &p, dock_ctx **out, std::string *err) {
    *out = nullptr;
    auto *c = new dock_ctx();
    c->params = p;
    c->device = rec->device;
    c->grid = rec->grid;
    c->rec = std::move(rec);
    auto bail = [&](const std::string &m) { *err = m; dock_free(c); return (int)DOCK_E_INTERNAL; };
    if (cudaSetDevice(c->device) != cudaSuccess) return bail("cudaSetDevice failed");
    {
        Trace tr("ctx.stream_create");
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail("cudaStreamCreate failed");
        if (cudaEventCreateWithFlags(&c->last_use, cudaEventDisableTiming) != cudaSuccess) return bail("cudaEventCreate failed");
    }
    {
        // kernel attributes are per device and process: set them once
        Trace tr("ctx.kernel_attributes");
        static std::mutex mu;
        static std::vector<int> done;
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(done.begin(), done.end(), c->device) == done.end()) {
            if (setup_kernel_attributes() != cudaSuccess) return bail("cudaFuncSetAttribute failed (is this an sm_100 device?)");
            done.push_back(c->device);
        }
    }
    Trace tr_rest("ctx.alloc_and_l2_window");
    if (dmalloc((void **)&c->d_dfs2orig, sizeof(int) * kMaxAtoms, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail("device allocation failed");
    if (p.l2_persist) {
        // NS: "Grid maps live in HBM with L2-persistence windows".
        // single attribute queries: cudaGetDeviceProperties is slow (all properties)
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
        if (max_persist > 0 && max_window > 0) {
            const size_t win = std::min(c->rec->bytes, (size_t)max_window);
            const size_t lim = std::min(win, (size_t)max_persist);
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            if (cur < lim) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);   // only ever grows
            cudaStreamAttrValue attr{};
            attr.accessPolicyWindow.base_ptr = c->rec->d_maps;
            attr.accessPolicyWindow.num_bytes = win;
            attr.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)lim / (double)win);
            attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
        }
        cudaGetLastError();   // the window is an optimisation: never fatal
    }
    *out = c;
    return DOCK_OK;
}

int ctx_reserve(dock_ctx *c, size_t blob_bytes, int runs, int pop) {
    CK(cudaSetDevice(c->device));
    CK(after_last_use(c, c->stream));   // the ligand block may still be read by an earlier call
    if (blob_bytes > c->blob_cap) {
        if (c->d_blob) { CK(cudaStreamSynchronize(c->stream)); dfree(c->d_blob, c->stream); }
        c->d_blob = nullptr; c->blob_cap = 0;
        CK(dmalloc((void **)&c->d_blob, blob_bytes, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->blob_cap = blob_bytes;
    }
    if (runs > 0 && pop > 0) return ensure_buffers(c, runs, pop);
    return DOCK_OK;
}

int ctx_attach_ligand(dock_ctx *c, Prepared &&p) {
    c->prep = std::move(p);
    if (int rc = ctx_reserve(c, c->prep.blob.size(), 0, 0)) return rc;
    CK(cudaMemcpyAsync(c->d_blob, c->prep.blob.data(), c->prep.blob.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_dfs2orig, c->prep.dfs2orig.data(), sizeof(int) * c->prep.N, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));   // host vectors may be reused by the caller
    c->lig = c->prep.layout;
    c->lig.blob = c->d_blob;
    return DOCK_OK;
}

}  // namespace dk

extern "C" {

int dock_params_default(dock_params *p) {
    if (!p) return DOCK_E_INPUT;
    std::memset(p, 0, sizeof(*p));
    p->p_tour = 0.60f; p->p_cross = 0.80f; p->p_mut = 0.02f; p->mut_trans = 2.0f; p->mut_angle = 0.523f;
    p->ls_method = DOCK_LS_ADADELTA; p->ls_rate = 1.0f; p->ls_max_iters = 300;
    p->sw_rho = 1.0f; p->sw_rho_min = 0.01f; p->sw_expand = 2.0f; p->sw_contract = 0.5f;
    p->sw_cons_succ = 4; p->sw_cons_fail = 4;
    p->ad_rho = 0.8f; p->ad_eps = 1e-2f;
    p->max_generations = 27000;
    p->device = 0; p->l2_persist = 1; p->gens_per_graph = 16;
    p->scoring = DOCK_SF_D5;   // AD4.1 coefficients (Huey et al. 2007), used by DOCK_SF_AD4
    p->w_vdw = 0.1662f; p->w_hb = 0.1209f; p->w_el = 0.1406f; p->w_ds = 0.1322f; p->w_tors = 0.2983f;
    p->qasp = 0.01097f;
    return DOCK_OK;
}

int dock_builtin_type_param(const char *name, dock_type_param *out) {
    static const struct { const char *n; dock_type_param t; } table[] = {
        {"C", {4.00f, 0.150f, -0.00143f, 33.5103f, 0}}, {"A", {4.00f, 0.150f, -0.00052f, 33.5103f, 0}},
        {"N", {3.50f, 0.160f, -0.00162f, 22.4493f, 0}}, {"NA", {3.50f, 0.160f, -0.00162f, 22.4493f, 2}},
        {"O", {3.20f, 0.200f, -0.00251f, 17.1573f, 0}}, {"OA", {3.20f, 0.200f, -0.00251f, 17.1573f, 2}},
        {"H", {2.00f, 0.020f, 0.00051f, 0.0f, 0}},      {"HD", {2.00f, 0.020f, 0.00051f, 0.0f, 1}},
    };
    if (!name || !out) return DOCK_E_INPUT;
    for (const auto &e : table)
        if (std::strcmp(e.n, name) == 0) { *out = e.t; return DOCK_OK; }
    return DOCK_E_INPUT;
}

int dock_init(const dock_grids *grids, const dock_type_param *type_params, const dock_ligand *ligand,
              const dock_params *params, dock_ctx **out) {
    if (!out) { g_init_error = "out: NULL"; return DOCK_E_INPUT; }
    *out = nullptr;
    dock_params p;
    if (params) p = *params; else dock_params_default(&p);
    std::string err;
    if (dk::validate_params(p, &err) != DOCK_OK) { g_init_error = err; return DOCK_E_INPUT; }
    std::vector<float4> packed;
    {
        Trace tr("init.pack_grid");
        if (dk::pack_grid(grids, &packed, &err) != DOCK_OK) { g_init_error = err; return DOCK_E_INPUT; }
    }
    std::vector<dock_type_param> tparams;
    if (dk::resolve_type_params(grids, type_params, &tparams, &err) != DOCK_OK) { g_init_error = err; return DOCK_E_INPUT; }
    dk::Prepared prep;
    {
        Trace tr("init.prepare_ligand");
        if (dk::prepare_ligand(ligand, tparams.data(), grids->n_types, dk::scoring_of(p), &prep, &err) != DOCK_OK) { g_init_error = err; return DOCK_E_INPUT; }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        g_init_error = "no CUDA device (this library has no CPU fallback)";
        return DOCK_E_INTERNAL;
    }
    if (p.device < 0 || p.device >= ndev) { g_init_error = "params.device: no such CUDA device"; return DOCK_E_INPUT; }
    std::shared_ptr<dk::Receptor> rec;
    {
        Trace tr("init.receptor_upload");
        if (int rc = dk::receptor_upload(grids, packed, p.device, &rec, &err)) { g_init_error = err; return rc; }
    }
    dock_ctx *c = nullptr;
    {
        Trace tr("init.ctx_create");
        if (int rc = dk::ctx_create(rec, p, &c, &err)) { g_init_error = err; return rc; }
    }
    Trace tr("init.attach_ligand");
    if (int rc = dk::ctx_attach_ligand(c, std::move(prep))) { g_init_error = c->err; dock_free(c); return rc; }
    *out = c;
    return DOCK_OK;
}

void dock_free(dock_ctx *c) {
    if (!c) return;
    Trace tr("free.total");
    cudaSetDevice(c->device);
    {
        Trace t1("free.sync");
        if (c->last_use) cudaEventSynchronize(c->last_use);   // kernels of asynchronous calls on other streams
        if (c->stream) cudaStreamSynchronize(c->stream);
    }
    {
        Trace t2("free.device_buffers");
        cudaStream_t s = c->stream;
        dk::dfree(c->d_blob, s); dk::dfree(c->d_dfs2orig, s);
        dk::dfree(c->d_genes, s); dk::dfree(c->d_E, s); dk::dfree(c->d_state, s); dk::dfree(c->d_perm, s);
        dk::dfree(c->d_ls_evals, s); dk::dfree(c->d_ls_count, s); dk::dfree(c->d_prof, s);
    }
    {
        Trace t3("free.events_and_stream");
        for (cudaEvent_t e : c->events) cudaEventDestroy(e);
        for (cudaEvent_t e : c->branch_events) cudaEventDestroy(e);
        for (cudaStream_t b : c->branch_streams) cudaStreamDestroy(b);
        if (c->last_use) cudaEventDestroy(c->last_use);
        if (c->stream) cudaStreamDestroy(c->stream);
    }
    cudaGetLastError();
    Trace t4("free.receptor_release");
    delete c;   // drops this context's reference to the receptor upload
}

const char *dock_last_error(const dock_ctx *c) { return c ? c->err.c_str() : g_init_error.c_str(); }
int dock_n_atoms(const dock_ctx *c) { return c ? c->prep.N : -1; }
int dock_n_torsions(const dock_ctx *c) { return c ? c->prep.T : -1; }
int dock_n_genes(const dock_ctx *c) { return c ? c->prep.G : -1; }
int dock_n_pairs(const dock_ctx *c) { return c ? c->prep.P : -1; }
int64_t dock_launch_count(const dock_ctx *c) { return c ? c->launches : -1; }

int dock_run_branches(const dock_ctx *c) { return c ? c->last_branches : -1; }
int dock_last_engine(const dock_ctx *c) { return c ? c->last_engine : -1; }
int dock_tile_schedule(const dock_ctx *c) {
    if (!c) return -1;
    const dk::LigDev &L = c->prep.layout;
    return (L.slot_mode ? 1 : 0) | (L.tail_rot ? 2 : 0) | (L.tail_seg && !((L.tail_seg >> 24) & 1) ? 4 : 0) |
           ((L.tail_seg >> 24) & 1 ? 8 : 0) | (L.packed ? 16 : 0) | ((L.nhb & 0xff) << 8);
}

int64_t dock_upload_bytes(const dock_ctx *c) {
    return c ? (int64_t)(c->rec->bytes + c->prep.blob.size() + sizeof(int) * c->prep.N) : -1;
}

int dock_kernel_stats(const dock_ctx *c, double *ms, int64_t *launches) {
    if (!c) return DOCK_E_INPUT;
    for (int i = 0; i < 3; ++i) {
        if (ms) ms[i] = c->prof_ms[i];
        if (launches) launches[i] = c->prof_n[i];
    }
    return DOCK_OK;
}

int dock_run_device(dock_ctx *c, int32_t pop, int32_t runs, int32_t run_base, uint32_t ligand_id, int64_t max_evals,
                    uint64_t seed, float *d_best_energy, float *d_best_genotype, int64_t *d_evals_used,
                    int32_t *d_generations, void *stream) {
    if (!c) return DOCK_E_INPUT;
    if (int rc = check_run_args(c, pop, runs, run_base, max_evals)) return rc;
    if (!d_best_energy || !d_best_genotype) return input_error(c, "d_best_energy/d_best_genotype: NULL");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_buffers(c, runs, pop)) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
    CK(dk::after_last_use(c, s));
    const dk::SearchDev sp = make_search(c, pop, runs, run_base, ligand_id, max_evals, seed);
    const dk::PopDev pd = pop_of(c);
    int K = c->params.gens_per_graph;
    if (sp.ls_method == DOCK_LS_ADADELTA || sp.n_ls == 0 || sp.ls_iters == 0) {
        // evaluations per generation are fixed (D10: exactly ls_iters per LS), so a short
        // job needs fewer captured generations than gens_per_graph (no trailing no-ops)
        const long long per_gen = (long long)(pop - 1) + (long long)sp.n_ls * sp.ls_iters;
        const long long need = per_gen > 0 ? (max_evals - pop + per_gen - 1) / per_gen : 1;
        K = (int)std::max(1LL, std::min<long long>(K, std::min<long long>(need, c->params.max_generations)));
    }
    // Run branches (dock_params.run_branches): with Solis-Wets the LS launch of a generation
    // lasts as long as its longest chain, so runs stepping together wait for the slowest of
    // all runs' chains every generation (1stp: max over 180 chains).  As independent graph
    // branches, each run waits only for its own chains; the termination poll stays per
    // graph batch.  ADADELTA chains all have the same length: lockstep (fewer launches).
    const bool do_ls = sp.n_ls > 0 && sp.ls_iters > 0;
    const int mode = c->params.run_branches;
    // Persistent clusters (k_run_sw): the whole Solis-Wets job in one launch,
    // one thread-block cluster per run looping over its generations on the device.
    if (do_ls && (mode == 3 || (mode == 0 && sp.ls_method == DOCK_LS_SOLIS_WETS)) && dk::run_sw_eligible(c->lig, sp)) {
        c->last_branches = runs;
        c->last_engine = 2;
        const bool prof = c->params.profile != 0;
        for (int i = 0; i < 3; ++i) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
        if (prof && !c->d_prof) CK(dk::dmalloc((void **)&c->d_prof, 2 * sizeof(unsigned long long), s));
        if (prof) CK(cudaMemsetAsync(c->d_prof, 0, 2 * sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(c->d_spec_done, 0, sizeof(unsigned) * (size_t)runs * 2 * pd.spec_words, s));
        CK(cudaMemsetAsync(c->d_spec_ctr, 0, sizeof(int) * (size_t)runs * 2, s));
        CK(dk::launch_init(c->lig, c->grid, sp, pd, s));
        CK(dk::launch_run_sw(c->lig, c->grid, sp, pd, prof ? c->d_prof : nullptr, s));
        CK(dk::launch_best(c->lig, sp, pd, d_best_energy, d_best_genotype, (long long *)d_evals_used, d_generations, s));
        CK(dk::mark_last_use(c, s));   // this path returns before k_run_sw finishes
        c->launches += 3;
        if (prof) {
            unsigned long long h[2] = {0, 0};
            CK(cudaMemcpyAsync(h, c->d_prof, sizeof h, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            c->prof_ms[1] = (double)h[0] * 1e-6; c->prof_n[1] = (long long)h[1];
        }
        return DOCK_OK;
    }
    // ADADELTA chains all last ls_max_iters iterations, so lockstep is best while one
    // generation's LS launch spans many waves; with few runs per GPU (the R split over 4-8
    // GPUs) the last partial wave idles most SMs and independent run branches fill it.
    // Measured on one B200, 7cpa: 13 runs 1.12e8 lockstep / 1.27e8 branches,
    // 25 runs 1.22e8 / 1.26e8, 50 runs 1.31e8 / 1.25e8, 100 runs 1.34e8 / 1.26e8.
    const bool ada_few = sp.ls_method == DOCK_LS_ADADELTA && do_ls &&
                         (long long)runs * sp.n_ls < 4LL * dk::adadelta_resident_groups(c->lig);
    const bool branched = runs > 1 && do_ls &&
                          (mode >= 2 || (mode == 0 && (sp.ls_method == DOCK_LS_SOLIS_WETS || ada_few)));
    const int NB = branched ? runs : 1;
    c->last_branches = NB;
    c->last_engine = branched ? 1 : 0;
    const bool prof = c->params.profile != 0;
    for (int i = 0; i < 3; ++i) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
    // events: lockstep 3 per generation (GA start, LS start, LS end) + 2 for init;
    // branched 2 per generation around run 0's LS node (every run's branch is the same
    // work; events on all branches, 2 x runs x K graph nodes, slowed 1stp 2.6x) + 2 for init
    const int n_ev = branched ? 2 * K + 2 : 3 * K + 2;
    const int ev_init = n_ev - 2;
    if (prof && (int)c->events.size() < n_ev) {
        while ((int)c->events.size() < n_ev) {
            cudaEvent_t ev;
            CK(cudaEventCreate(&ev));
            c->events.push_back(ev);
        }
    }
    if (branched) {
        while ((int)c->branch_streams.size() < NB) {
            cudaStream_t b;
            CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
            c->branch_streams.push_back(b);
        }
        while ((int)c->branch_events.size() < NB + 1) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->branch_events.push_back(e);
        }
    }
    cudaEvent_t *ev = c->events.data();
    if (prof) CK(cudaEventRecord(ev[ev_init], s));
    CK(dk::launch_init(c->lig, c->grid, sp, pd, s));
    if (prof) CK(cudaEventRecord(ev[ev_init + 1], s));
    c->launches += 1;
    dk::LsArgs la{};
    la.use_state = 1; la.n_per_run = sp.n_ls; la.iters = sp.ls_iters;
    la.wave_total = runs * sp.n_ls;      // the speculation-depth rule sees every run's chains
    // capture K generations once; the kernels read the generation from device state
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    auto t_cap = std::chrono::steady_clock::now();
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaError_t ce = cudaSuccess;
    if (!branched) {
        for (int k = 0; k < K && ce == cudaSuccess; ++k) {
            // profile 1: events around the LS node only (2 graph nodes per generation);
            // profile 2: also around the GA node
            if (prof && c->params.profile >= 2) ce = cudaEventRecordWithFlags(ev[3 * k], s, cudaEventRecordExternal);
            if (ce == cudaSuccess) ce = dk::launch_ga(c->lig, c->grid, sp, pd, nullptr, s);
            if (ce == cudaSuccess && prof) ce = cudaEventRecordWithFlags(ev[3 * k + 1], s, cudaEventRecordExternal);
            if (ce == cudaSuccess && do_ls) ce = dk::launch_ls(c->lig, c->grid, sp, pd, la, runs * sp.n_ls, s);
            if (ce == cudaSuccess && prof) ce = cudaEventRecordWithFlags(ev[3 * k + 2], s, cudaEventRecordExternal);
            if (ce == cudaSuccess && !do_ls) ce = dk::launch_gen_end(sp, pd, s);   // else fused into k_ls_*
        }
    } else {
        // fork: every run's K generations on its own stream, on a one-run view of the
        // population buffers (rstride keeps the parity blocks' stride), then join
        const size_t G = (size_t)c->prep.G, P = (size_t)pop;
        ce = cudaEventRecord(c->branch_events[0], s);
        for (int r = 0; r < NB && ce == cudaSuccess; ++r) {
            cudaStream_t b = c->branch_streams[r];
            ce = cudaStreamWaitEvent(b, c->branch_events[0], 0);
            dk::SearchDev spr = sp;
            spr.runs = 1; spr.run_base = sp.run_base + r;
            dk::PopDev pr = pd;
            pr.genes = pd.genes + (size_t)r * P * G; pr.E = pd.E + (size_t)r * P; pr.state = pd.state + r;
            pr.perm = pd.perm + (size_t)r * P; pr.ls_evals = pd.ls_evals + (size_t)r * P;
            pr.ls_count = pd.ls_count + r;
            pr.spec_done = pd.spec_done + (size_t)r * 2 * pd.spec_words; pr.spec_ctr = pd.spec_ctr + 2 * r;
            for (int k = 0; k < K && ce == cudaSuccess; ++k) {
                ce = dk::launch_ga(c->lig, c->grid, spr, pr, nullptr, b);
                if (ce == cudaSuccess && prof && r == 0) ce = cudaEventRecordWithFlags(ev[2 * k], b, cudaEventRecordExternal);
                if (ce == cudaSuccess) ce = dk::launch_ls(c->lig, c->grid, spr, pr, la, sp.n_ls, b);
                if (ce == cudaSuccess && prof && r == 0) ce = cudaEventRecordWithFlags(ev[2 * k + 1], b, cudaEventRecordExternal);
            }
            if (ce == cudaSuccess) ce = cudaEventRecord(c->branch_events[1 + r], b);
            if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, c->branch_events[1 + r], 0);
        }
    }
    cudaError_t ee = cudaStreamEndCapture(s, &graph);
    if (ce != cudaSuccess || ee != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        c->err = std::string("graph capture: ") + cudaGetErrorString(ce != cudaSuccess ? ce : ee);
        return DOCK_E_INTERNAL;
    }
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        cudaGraphDestroy(graph);
        c->err = "cudaGraphInstantiate failed";
        return DOCK_E_INTERNAL;
    }
    if (Trace::on())
        std::fprintf(stderr, "[dock] run.graph_capture+instantiate %.3f ms (%d branches)\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_cap).count(), NB);
    const int per_graph = NB * K * 2;   // GA + LS (gen end fused), or GA + gen end
    const long long max_batches = (long long)c->params.max_generations / K + 2;
    int rc = DOCK_OK;
    for (long long b = 0; b < max_batches; ++b) {
        cudaError_t e = cudaGraphLaunch(exec, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(c->h_state.data(), c->d_state, sizeof(dk::RunState) * runs, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { c->err = std::string("generation batch: ") + cudaGetErrorString(e); rc = DOCK_E_INTERNAL; break; }
        c->launches += per_graph;
        if (prof) {
            float t;
            cudaError_t pe = cudaSuccess;
            if (b == 0 && (pe = cudaEventElapsedTime(&t, ev[ev_init], ev[ev_init + 1])) == cudaSuccess) { c->prof_ms[2] += t; c->prof_n[2] += 1; }
            if (branched) {
                for (int q = 0; q < K && pe == cudaSuccess; ++q)
                    if ((pe = cudaEventElapsedTime(&t, ev[2 * q], ev[2 * q + 1])) == cudaSuccess) { c->prof_ms[1] += t; c->prof_n[1] += 1; }
            } else {
                for (int k = 0; k < K && pe == cudaSuccess; ++k) {
                    if (c->params.profile >= 2 && (pe = cudaEventElapsedTime(&t, ev[3 * k], ev[3 * k + 1])) == cudaSuccess) { c->prof_ms[0] += t; c->prof_n[0] += 1; }
                    if (pe == cudaSuccess && do_ls && (pe = cudaEventElapsedTime(&t, ev[3 * k + 1], ev[3 * k + 2])) == cudaSuccess) { c->prof_ms[1] += t; c->prof_n[1] += 1; }
                }
            }
            if (pe != cudaSuccess) {
                c->err = std::string("profiling (ignored): cudaEventElapsedTime: ") + cudaGetErrorString(pe);
                cudaGetLastError();
                c->prof_n[0] = c->prof_n[1] = -1;
            }
        }
        bool any = false;
        for (int r = 0; r < runs && !any; ++r)
            any = c->h_state[r].evals < max_evals && c->h_state[r].gen < c->params.max_generations;
        if (!any) break;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (rc != DOCK_OK) return rc;
    CK(dk::launch_best(c->lig, sp, pd, d_best_energy, d_best_genotype, (long long *)d_evals_used, d_generations, s));
    CK(dk::mark_last_use(c, s));
    c->launches += 1;
    return DOCK_OK;
}

int dock_run_ex(dock_ctx *c, int32_t pop, int32_t runs, int32_t run_base, uint32_t ligand_id, int64_t max_evals,
                uint64_t seed, float *best_energy, float *best_genotype, float *best_xyz, int64_t *evals_used,
                int32_t *generations) {
    if (!c) return DOCK_E_INPUT;
    if (int rc = check_run_args(c, pop, runs, run_base, max_evals)) return rc;
    if (!best_energy || !best_genotype) return input_error(c, "best_energy/best_genotype: NULL");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G, N = c->prep.N;
    DevBuf bE(c->stream), bG(c->stream), bEv(c->stream), bGen(c->stream), bX(c->stream), bE2(c->stream);
    CK(bE.alloc(sizeof(float) * runs));
    CK(bG.alloc(sizeof(float) * runs * G));
    CK(bEv.alloc(sizeof(int64_t) * runs));
    CK(bGen.alloc(sizeof(int32_t) * runs));
    int rc = dock_run_device(c, pop, runs, run_base, ligand_id, max_evals, seed, (float *)bE.p, (float *)bG.p,
                             (int64_t *)bEv.p, (int32_t *)bGen.p, c->stream);
    if (rc != DOCK_OK) return rc;
    if (best_xyz) {
        CK(bX.alloc(sizeof(float) * runs * N * 3));
        CK(bE2.alloc(sizeof(float) * runs));
        CK(dk::launch_eval(c->lig, c->grid, runs, (const float *)bG.p, (float *)bE2.p, nullptr, (float *)bX.p,
                           c->d_dfs2orig, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(best_xyz, bX.p, sizeof(float) * runs * N * 3, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaMemcpyAsync(best_energy, bE.p, sizeof(float) * runs, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(best_genotype, bG.p, sizeof(float) * runs * G, cudaMemcpyDeviceToHost, c->stream));
    if (evals_used) CK(cudaMemcpyAsync(evals_used, bEv.p, sizeof(int64_t) * runs, cudaMemcpyDeviceToHost, c->stream));
    if (generations) CK(cudaMemcpyAsync(generations, bGen.p, sizeof(int32_t) * runs, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DOCK_OK;
}

int dock_run(dock_ctx *c, int32_t pop, int32_t runs, int64_t max_evals, uint64_t seed, float *best_energy,
             float *best_genotype, float *best_xyz, int64_t *evals_used, int32_t *generations) {
    return dock_run_ex(c, pop, runs, 0, 0u, max_evals, seed, best_energy, best_genotype, best_xyz, evals_used,
                       generations);
}

int dock_eval_device(dock_ctx *c, int32_t n, const float *d_genotypes, float *d_energy, float *d_grad, float *d_xyz,
                     void *stream) {
    if (!c) return DOCK_E_INPUT;
    if (n < 0) return input_error(c, "n: must be >= 0");
    if (n > 0 && (!d_genotypes || !d_energy)) return input_error(c, "d_genotypes/d_energy: NULL");
    CK(cudaSetDevice(c->device));
    CK(dk::after_last_use(c, (cudaStream_t)stream));
    CK(dk::launch_eval(c->lig, c->grid, n, d_genotypes, d_energy, d_grad, d_xyz, c->d_dfs2orig, (cudaStream_t)stream));
    CK(dk::mark_last_use(c, (cudaStream_t)stream));
    c->launches += 1;
    return DOCK_OK;
}

int dock_bench_part(dock_ctx *c, int32_t part, int32_t n, int32_t iters, const float *d_genotypes, float *d_out,
                    void *stream) {
    if (!c) return DOCK_E_INPUT;
    if (part < 0 || part > 1 || n < 0 || iters < 1) return input_error(c, "part in {0,1}, n >= 0, iters >= 1");
    if (n > 0 && (!d_genotypes || !d_out)) return input_error(c, "d_genotypes/d_out: NULL");
    CK(cudaSetDevice(c->device));
    CK(dk::after_last_use(c, (cudaStream_t)stream));
    CK(dk::launch_bench_part(c->lig, c->grid, part, n, iters, d_genotypes, d_out, (cudaStream_t)stream));
    CK(dk::mark_last_use(c, (cudaStream_t)stream));
    c->launches += 1;
    return DOCK_OK;
}

int dock_eval(dock_ctx *c, int32_t n, const float *genotypes, float *energy, float *grad, float *xyz) {
    if (!c) return DOCK_E_INPUT;
    if (n < 0) return input_error(c, "n: must be >= 0");
    if (n == 0) return DOCK_OK;
    if (!genotypes || !energy) return input_error(c, "genotypes/energy: NULL");
    for (long long i = 0; i < (long long)n * c->prep.G; ++i)
        if (!std::isfinite(genotypes[i])) return input_error(c, "genotypes[" + std::to_string(i) + "]: non-finite");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G, N = c->prep.N;
    DevBuf dg(c->stream), dE(c->stream), dgr(c->stream), dx(c->stream);
    CK(dg.alloc(sizeof(float) * n * G));
    CK(dE.alloc(sizeof(float) * n));
    if (grad) CK(dgr.alloc(sizeof(float) * n * G));
    if (xyz) CK(dx.alloc(sizeof(float) * n * N * 3));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(dg.p, genotypes, sizeof(float) * n * G, cudaMemcpyHostToDevice, c->stream));
    CK(dk::launch_eval(c->lig, c->grid, n, (const float *)dg.p, (float *)dE.p, (float *)dgr.p, (float *)dx.p,
                       c->d_dfs2orig, c->stream));
    c->launches += 1;
    CK(cudaMemcpyAsync(energy, dE.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (grad) CK(cudaMemcpyAsync(grad, dgr.p, sizeof(float) * n * G, cudaMemcpyDeviceToHost, c->stream));
    if (xyz) CK(cudaMemcpyAsync(xyz, dx.p, sizeof(float) * n * N * 3, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DOCK_OK;
}

int dock_eval_terms(dock_ctx *c, int32_t n, const float *genotypes, float *inter, float *intra, float *dG) {
    if (!c) return DOCK_E_INPUT;
    if (n < 0) return input_error(c, "n: must be >= 0");
    if (n == 0) return DOCK_OK;
    if (!genotypes) return input_error(c, "genotypes: NULL");
    for (long long i = 0; i < (long long)n * c->prep.G; ++i)
        if (!std::isfinite(genotypes[i])) return input_error(c, "genotypes[" + std::to_string(i) + "]: non-finite");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G;
    DevBuf dg(c->stream), dI(c->stream), dP(c->stream);
    CK(dg.alloc(sizeof(float) * n * G));
    CK(dI.alloc(sizeof(float) * n));
    CK(dP.alloc(sizeof(float) * n));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(dg.p, genotypes, sizeof(float) * n * G, cudaMemcpyHostToDevice, c->stream));
    CK(dk::launch_eval(c->lig, c->grid, n, (const float *)dg.p, (float *)dI.p, nullptr, nullptr, c->d_dfs2orig,
                       c->stream, dk::kPartsInter));
    CK(dk::launch_eval(c->lig, c->grid, n, (const float *)dg.p, (float *)dP.p, nullptr, nullptr, c->d_dfs2orig,
                       c->stream, dk::kPartsIntra));
    c->launches += 2;
    std::vector<float> hi(n);
    CK(cudaMemcpyAsync(hi.data(), dI.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (intra) CK(cudaMemcpyAsync(intra, dP.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (inter) std::copy(hi.begin(), hi.end(), inter);
    // AD4 binding estimate: inter + w_tors * T (host: one multiply-add per genotype)
    const float w_tors = c->params.scoring == DOCK_SF_AD4 ? c->params.w_tors : 0.0f;
    if (dG) for (int i = 0; i < n; ++i) dG[i] = hi[i] + w_tors * (float)c->prep.T;
    return DOCK_OK;
}

int dock_cluster(dock_ctx *c, int32_t n, const float *xyz, const float *energy, float rmsd_tol, int32_t *cluster,
                 float *rmsd_to_seed, int32_t *rank, int32_t *n_clusters) {
    if (!c) return DOCK_E_INPUT;
    if (!n_clusters) return input_error(c, "n_clusters: NULL");
    if (n < 0 || n > dk::kClusterMaxPoses) return input_error(c, "n: must be in 0..4096");
    if (n == 0) { *n_clusters = 0; return DOCK_OK; }
    if (!xyz || !energy || !cluster || !rmsd_to_seed) return input_error(c, "xyz/energy/cluster/rmsd_to_seed: NULL");
    if (!std::isfinite(rmsd_tol) || rmsd_tol < 0.f) return input_error(c, "rmsd_tol: must be finite and >= 0");
    const int N = c->prep.N;
    for (long long i = 0; i < (long long)n * N * 3; ++i)
        if (!std::isfinite(xyz[i])) return input_error(c, "xyz[" + std::to_string(i) + "]: non-finite");
    CK(cudaSetDevice(c->device));
    DevBuf dx(c->stream), dE(c->stream), dc(c->stream), dr(c->stream), dk_(c->stream), dn(c->stream);
    CK(dx.alloc(sizeof(float) * n * N * 3));
    CK(dE.alloc(sizeof(float) * n));
    CK(dc.alloc(sizeof(int) * n));
    CK(dr.alloc(sizeof(float) * n));
    CK(dk_.alloc(sizeof(int) * n));
    CK(dn.alloc(sizeof(int)));
    CK(cudaMemcpyAsync(dx.p, xyz, sizeof(float) * n * N * 3, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dE.p, energy, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
    CK(dk::launch_cluster(n, N, (const float *)dx.p, (const float *)dE.p, rmsd_tol, (int *)dc.p, (float *)dr.p,
                          (int *)dk_.p, (int *)dn.p, c->stream));
    c->launches += 1;
    CK(cudaMemcpyAsync(cluster, dc.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(rmsd_to_seed, dr.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (rank) CK(cudaMemcpyAsync(rank, dk_.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(n_clusters, dn.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DOCK_OK;
}

int dock_bench_l2_gather(int32_t device, int32_t mib, int32_t blocks_per_sm, int32_t iters, double *gbps, double *ms) {
    if (mib < 1 || mib > 4096 || blocks_per_sm < 1 || iters < 1 || !gbps) {
        g_init_error = "bench_l2_gather: mib 1..4096, blocks_per_sm >= 1, iters >= 1, gbps non-NULL";
        return DOCK_E_INPUT;
    }
    dock_ctx tmp;
    dock_ctx *c = &tmp;
    c->device = device;
    CK(cudaSetDevice(device));
    int nsm = 148;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const size_t n = (size_t)mib * (1u << 20) / 16;
    DevBuf buf(c->stream), out(c->stream);
    CK(buf.alloc(n * 16));
    CK(out.alloc((size_t)nsm * blocks_per_sm * 256 * 4));
    CK(cudaMemsetAsync(buf.p, 0, n * 16, c->stream));
    const int blocks = nsm * blocks_per_sm;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(dk::launch_l2_gather((const float4 *)buf.p, (uint32_t)n, blocks, iters, (float *)out.p, c->stream));   // warm-up
    CK(cudaEventRecord(e0, c->stream));
    CK(dk::launch_l2_gather((const float4 *)buf.p, (uint32_t)n, blocks, iters, (float *)out.p, c->stream));
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    *gbps = 16.0 * 8.0 * (double)blocks * 256 * iters / (t * 1e-3) / 1e9;
    if (ms) *ms = t;
    return DOCK_OK;
}

int dock_topology(const dock_ligand *ligand, const dock_type_param *type_params, int32_t n_types, int32_t *n_tors,
                  int32_t *axis, uint8_t *moved, int32_t *n_pairs, int32_t *pairs, int32_t pair_cap) {
    dk::Prepared p;
    std::string err;
    if (dk::prepare_ligand(ligand, type_params, n_types, dk::Scoring(), &p, &err) != DOCK_OK) { g_init_error = err; return DOCK_E_INPUT; }
    if (n_tors) *n_tors = p.T;
    if (n_pairs) *n_pairs = p.P;
    for (int k = 0; k < p.T; ++k)
        if (axis) { axis[2 * k] = p.tor_a[k]; axis[2 * k + 1] = p.tor_b[k]; }
    if (moved) std::copy(p.moved.begin(), p.moved.end(), moved);
    if (pairs) {
        if (p.P > pair_cap) { g_init_error = "pair_cap: too small"; return DOCK_E_INPUT; }
        std::copy(p.pairs.begin(), p.pairs.end(), pairs);
    }
    return DOCK_OK;
}

int dock_get_pairs(const dock_ctx *c, int32_t *pairs) {
    if (!c || !pairs) return DOCK_E_INPUT;
    std::copy(c->prep.pairs.begin(), c->prep.pairs.end(), pairs);
    return DOCK_OK;
}

int dock_get_torsions(const dock_ctx *c, int32_t *axis, uint8_t *moved) {
    if (!c) return DOCK_E_INPUT;
    for (int k = 0; k < c->prep.T; ++k) {
        if (axis) { axis[2 * k] = c->prep.tor_a[k]; axis[2 * k + 1] = c->prep.tor_b[k]; }
    }
    if (moved) std::copy(c->prep.moved.begin(), c->prep.moved.end(), moved);
    return DOCK_OK;
}

int dock_philox(int32_t n, const uint32_t *ctr4, const uint32_t *key2, uint32_t *out4) {
    if (n < 0 || (n > 0 && (!ctr4 || !key2 || !out4))) return DOCK_E_INPUT;
    if (n == 0) return DOCK_OK;
    dock_ctx tmp;
    dock_ctx *c = &tmp;
    DevBuf dc(c->stream), dk_(c->stream), dout(c->stream);
    CK(dc.alloc(16 * (size_t)n));
    CK(dk_.alloc(8 * (size_t)n));
    CK(dout.alloc(16 * (size_t)n));
    CK(cudaMemcpy(dc.p, ctr4, 16 * (size_t)n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dk_.p, key2, 8 * (size_t)n, cudaMemcpyHostToDevice));
    CK(dk::launch_philox(n, (const uint32_t *)dc.p, (const uint32_t *)dk_.p, (uint32_t *)dout.p, nullptr));
    CK(cudaMemcpy(out4, dout.p, 16 * (size_t)n, cudaMemcpyDeviceToHost));
    return DOCK_OK;
}

int dock_stream_words(uint64_t seed, uint32_t ligand_id, uint32_t purpose, uint32_t slot, uint32_t gen, uint32_t run,
                      uint32_t m0, int32_t n, uint32_t *out) {
    if (n < 0 || (n > 0 && !out) || purpose > 255 || slot >= (1u << 24)) return DOCK_E_INPUT;
    if (n == 0) return DOCK_OK;
    dock_ctx tmp;
    dock_ctx *c = &tmp;
    const uint64_t k = seed + (uint64_t)ligand_id * 0x9E3779B97F4A7C15ull;
    DevBuf d(c->stream);
    CK(d.alloc(4 * (size_t)n));
    CK(dk::launch_stream_words((uint32_t)k, (uint32_t)(k >> 32), purpose, slot, gen, run, m0, n, (uint32_t *)d.p, nullptr));
    CK(cudaMemcpy(out, d.p, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    return DOCK_OK;
}

int dock_init_population(dock_ctx *c, int32_t pop, int32_t runs, int32_t run_base, uint32_t ligand_id, uint64_t seed,
                         float *genes, float *energy) {
    if (!c) return DOCK_E_INPUT;
    if (int rc = check_run_args(c, pop, runs, run_base, pop)) return rc;
    if (!genes || !energy) return input_error(c, "genes/energy: NULL");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_buffers(c, runs, pop)) return rc;
    CK(dk::after_last_use(c, c->stream));
    const dk::SearchDev sp = make_search(c, pop, runs, run_base, ligand_id, pop, seed);
    CK(dk::launch_init(c->lig, c->grid, sp, pop_of(c), c->stream));
    c->launches += 1;
    const size_t G = (size_t)c->prep.G;   // generation 0 is parity block 0, rows [run][pop][G]
    CK(cudaMemcpyAsync(genes, c->d_genes, sizeof(float) * runs * pop * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(energy, c->d_E, sizeof(float) * runs * pop, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DOCK_OK;
}

int dock_ga_step(dock_ctx *c, uint64_t seed, uint32_t ligand_id, int32_t run, int32_t gen, int32_t pop,
                 const float *old_genes, const float *old_E, float *new_genes, float *new_E, int32_t *debug,
                 int32_t *perm) {
    if (!c) return DOCK_E_INPUT;
    if (pop < 2 || pop > 4096) return input_error(c, "pop: must be in 2..4096");
    if (gen < 1 || run < 0) return input_error(c, "gen >= 1 and run >= 0 required");
    if (!old_genes || !old_E || !new_genes || !new_E) return input_error(c, "ga_step buffers: NULL");
    CK(cudaSetDevice(c->device));
    if (int rc = ensure_buffers(c, 1, pop)) return rc;
    const int G = c->prep.G;
    dk::SearchDev sp = make_search(c, pop, 1, run, ligand_id, LLONG_MAX, seed);
    sp.max_generations = INT_MAX;
    const dk::PopDev pd = pop_of(c);
    const int cur = (gen - 1) & 1, nxt = gen & 1;
    dk::RunState st{0, gen - 1, 0};
    DevBuf ddbg(c->stream);
    CK(ddbg.alloc(sizeof(int) * 8 * pop));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(c->d_genes + (size_t)cur * 1 * pop * G, old_genes, sizeof(float) * pop * G, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_E + (size_t)cur * pop, old_E, sizeof(float) * pop, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_state, &st, sizeof(st), cudaMemcpyHostToDevice, c->stream));
    CK(dk::launch_ga(c->lig, c->grid, sp, pd, (int *)ddbg.p, c->stream));
    c->launches += 1;
    CK(cudaMemcpyAsync(new_genes, c->d_genes + (size_t)nxt * pop * G, sizeof(float) * pop * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(new_E, c->d_E + (size_t)nxt * pop, sizeof(float) * pop, cudaMemcpyDeviceToHost, c->stream));
    if (debug) CK(cudaMemcpyAsync(debug, ddbg.p, sizeof(int) * 8 * pop, cudaMemcpyDeviceToHost, c->stream));
    if (perm) CK(cudaMemcpyAsync(perm, c->d_perm, sizeof(int) * pop, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DOCK_OK;
}

int dock_sw_trace(dock_ctx *c, int32_t n, int32_t iters, uint64_t seed, uint32_t ligand_id, int32_t run, int32_t gen,
                  const int32_t *slots, const float *fed_energy, float *genes, float *energy, int64_t *evals,
                  int32_t *trace_outcome, float *trace_rho) {
    if (!c) return DOCK_E_INPUT;
    if (n < 0 || iters < 0) return input_error(c, "n, iters: must be >= 0");
    if (n == 0 || iters == 0) return DOCK_OK;
    if (!slots || !genes || !energy || !trace_outcome || !trace_rho) return input_error(c, "sw_trace buffers: NULL");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G;
    dk::SearchDev sp = make_search(c, 2, 1, run, ligand_id, LLONG_MAX, seed);
    sp.ls_method = DOCK_LS_SOLIS_WETS;
    const size_t nt = (size_t)n * iters;
    DevBuf dg(c->stream), dE(c->stream), dev(c->stream), dsl(c->stream), dfed(c->stream), dtr(c->stream),
        drho(c->stream);
    CK(dg.alloc(sizeof(float) * n * G));
    CK(dE.alloc(sizeof(float) * n));
    CK(dev.alloc(sizeof(int) * n));
    CK(dsl.alloc(sizeof(int) * n));
    CK(dtr.alloc(sizeof(int) * nt));
    CK(drho.alloc(sizeof(float) * nt));
    if (fed_energy) CK(dfed.alloc(sizeof(float) * nt * 2));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(dg.p, genes, sizeof(float) * n * G, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dE.p, energy, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dsl.p, slots, sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    if (fed_energy) CK(cudaMemcpyAsync(dfed.p, fed_energy, sizeof(float) * nt * 2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(dtr.p, 0xff, sizeof(int) * nt, c->stream));   // -1: not executed
    CK(cudaMemsetAsync(drho.p, 0, sizeof(float) * nt, c->stream));
    dk::LsArgs la{};
    la.use_state = 0; la.n_per_run = n; la.iters = iters;
    la.genes = (float *)dg.p; la.E = (float *)dE.p; la.evals = (int *)dev.p; la.rng_slot = (const int *)dsl.p;
    la.gen = gen; la.run = run;
    la.sw_fed = (const float *)dfed.p; la.sw_trace = (int *)dtr.p; la.sw_trace_rho = (float *)drho.p;
    CK(dk::launch_ls(c->lig, c->grid, sp, pop_of(c), la, n, c->stream));
    c->launches += 1;
    std::vector<int> ev(n);
    CK(cudaMemcpyAsync(genes, dg.p, sizeof(float) * n * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(energy, dE.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(ev.data(), dev.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(trace_outcome, dtr.p, sizeof(int) * nt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(trace_rho, drho.p, sizeof(float) * nt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (evals) for (int i = 0; i < n; ++i) evals[i] = ev[i];
    return DOCK_OK;
}

int dock_ad_trace(dock_ctx *c, int32_t n, int32_t iters, const float *fed, float *genes, float *energy, int64_t *evals,
                  float *trace_x, float *trace_E, float *trace_g) {
    if (!c) return DOCK_E_INPUT;
    if (n < 0 || iters < 0) return input_error(c, "n, iters: must be >= 0");
    if (n == 0 || iters == 0) return DOCK_OK;
    if (!genes || !energy || !trace_x || !trace_E || !trace_g) return input_error(c, "ad_trace buffers: NULL");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G;
    dk::SearchDev sp = make_search(c, 2, 1, 0, 0, LLONG_MAX, 0);
    sp.ls_method = DOCK_LS_ADADELTA;
    const size_t nt = (size_t)n * iters;
    DevBuf dg(c->stream), dE(c->stream), dev(c->stream), dsl(c->stream), dfed(c->stream), dtx(c->stream),
        dtE(c->stream), dtg(c->stream);
    CK(dg.alloc(sizeof(float) * n * G));
    CK(dE.alloc(sizeof(float) * n));
    CK(dev.alloc(sizeof(int) * n));
    CK(dsl.alloc(sizeof(int) * n));
    CK(dtx.alloc(sizeof(float) * nt * G));
    CK(dtE.alloc(sizeof(float) * nt));
    CK(dtg.alloc(sizeof(float) * nt * G));
    if (fed) CK(dfed.alloc(sizeof(float) * nt * (G + 1)));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(dg.p, genes, sizeof(float) * n * G, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dE.p, energy, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(dsl.p, 0, sizeof(int) * n, c->stream));
    if (fed) CK(cudaMemcpyAsync(dfed.p, fed, sizeof(float) * nt * (G + 1), cudaMemcpyHostToDevice, c->stream));
    dk::LsArgs la{};
    la.use_state = 0; la.n_per_run = n; la.iters = iters;
    la.genes = (float *)dg.p; la.E = (float *)dE.p; la.evals = (int *)dev.p; la.rng_slot = (const int *)dsl.p;
    la.gen = 1; la.run = 0;
    la.ad_fed = (const float *)dfed.p;
    la.ad_trace_x = (float *)dtx.p; la.ad_trace_E = (float *)dtE.p; la.ad_trace_g = (float *)dtg.p;
    CK(dk::launch_ls(c->lig, c->grid, sp, pop_of(c), la, n, c->stream));
    c->launches += 1;
    std::vector<int> ev(n);
    CK(cudaMemcpyAsync(genes, dg.p, sizeof(float) * n * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(energy, dE.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(ev.data(), dev.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(trace_x, dtx.p, sizeof(float) * nt * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(trace_E, dtE.p, sizeof(float) * nt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(trace_g, dtg.p, sizeof(float) * nt * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (evals) for (int i = 0; i < n; ++i) evals[i] = ev[i];
    return DOCK_OK;
}

int dock_ls_step(dock_ctx *c, int32_t method, int32_t n, int32_t iters, uint64_t seed, uint32_t ligand_id,
                 int32_t run, int32_t gen, const int32_t *slots, float *genes, float *energy, int64_t *evals) {
    if (!c) return DOCK_E_INPUT;
    if (method != DOCK_LS_ADADELTA && method != DOCK_LS_SOLIS_WETS) return input_error(c, "method: 0 or 1");
    if (n < 0 || iters < 0) return input_error(c, "n, iters: must be >= 0");
    if (n == 0) return DOCK_OK;
    if (!slots || !genes || !energy) return input_error(c, "ls_step buffers: NULL");
    CK(cudaSetDevice(c->device));
    const int G = c->prep.G;
    dk::SearchDev sp = make_search(c, 2, 1, run, ligand_id, LLONG_MAX, seed);
    sp.ls_method = method;
    DevBuf dg(c->stream), dE(c->stream), dev(c->stream), dsl(c->stream);
    CK(dg.alloc(sizeof(float) * n * G));
    CK(dE.alloc(sizeof(float) * n));
    CK(dev.alloc(sizeof(int) * n));
    CK(dsl.alloc(sizeof(int) * n));
    CK(dk::after_last_use(c, c->stream));
    CK(cudaMemcpyAsync(dg.p, genes, sizeof(float) * n * G, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dE.p, energy, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dsl.p, slots, sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    dk::LsArgs la{};
    la.use_state = 0; la.n_per_run = n; la.iters = iters;
    la.genes = (float *)dg.p; la.E = (float *)dE.p; la.evals = (int *)dev.p; la.rng_slot = (const int *)dsl.p;
    la.gen = gen; la.run = run;
    CK(dk::launch_ls(c->lig, c->grid, sp, pop_of(c), la, n, c->stream));
    c->launches += 1;
    std::vector<int> ev(n);
    CK(cudaMemcpyAsync(genes, dg.p, sizeof(float) * n * G, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(energy, dE.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(ev.data(), dev.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (evals) for (int i = 0; i < n; ++i) evals[i] = ev[i];
    return DOCK_OK;
}

}  // extern "C"
