// screen.cpp — dock_screen: many ligands against one receptor on one or more GPUs (row
// "multi-GPU ligand scheduler" of SURVEY.md §8(e); PAPER.md:34-38 [§I]: docking a library
// is "a load balancing and dataflow execution optimization problem" over heterogeneous
// ligands; runs are independent).
//
// Design (one process, several devices; the torch.distributed rank sharding in
// paper_2203_02096_b200/sched.py sits above this for one-process-per-GPU launches):
//   1. host preprocessing (D1 + constant block) of every ligand on a thread pool;
//   2. longest-processing-time-first order by the §8(e) cost model 40 P + 133 N (every
//      ligand of a screen has the same runs x max_evals, so that factor drops out);
//   3. one receptor upload per device, shared by `slots` engine contexts per device, each
//      with its own stream, so several ligands are in flight per GPU and their kernels
//      fill the 148 SMs together (one C4 ligand alone is ~1,500 lane groups);
//   4. one worker thread per slot pulls the next ligand from a shared atomic cursor
//      (dynamic LPT: the longest remaining ligand goes to the first free slot);
//   5. per ligand: dock_run_device on the slot's stream, 4 B + 4 B + G*4 B per run back
//      to host memory, best over runs on the host (lowest run on ties).
// A ligand's result depends only on (inputs, seed, ligand_id): the Philox key is
// seed + ligand_id * 0x9E3779B97F4A7C15 (D2), never the slot or the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"

namespace {

thread_local std::string g_screen_error;

struct SlotBufs {
    float *d_bE = nullptr, *d_bG = nullptr;
    int64_t *d_ev = nullptr;
    dk::PinnedBuf<float> h_bE, h_bG;
    dk::PinnedBuf<int64_t> h_ev;
    void release(cudaStream_t s) {
        dk::dfree(d_bE, s); dk::dfree(d_bG, s); dk::dfree(d_ev, s);
        d_bE = d_bG = nullptr; d_ev = nullptr;
    }
};

}  // namespace

extern "C" int dock_screen(const dock_grids *grids, const dock_type_param *type_params, const dock_ligand *ligands,
                           int32_t n_ligands, const uint32_t *ligand_ids, const dock_params *params,
                           const dock_screen_opts *opts, int32_t pop, int32_t runs, int64_t max_evals, uint64_t seed,
                           float *best_energy, int32_t *best_run, float *best_genotype, int64_t *evals_used,
                           int32_t *status, int32_t *device_of, dock_screen_stats *stats) {
    using clk = std::chrono::steady_clock;
    auto fail_input = [](const std::string &m) { g_screen_error = m; return (int)DOCK_E_INPUT; };
    if (n_ligands < 0) return fail_input("n_ligands: must be >= 0");
    if (n_ligands > 0 && (!ligands || !best_energy || !best_genotype)) return fail_input("ligands/best_energy/best_genotype: NULL");
    std::vector<dock_type_param> tparams;
    {
        std::string terr;
        if (dk::resolve_type_params(grids, type_params, &tparams, &terr) != DOCK_OK) return fail_input(terr);
    }
    type_params = tparams.data();   // per-type parameters by value, or the built-in table by name
    if (pop < 2 || pop > 4096) return fail_input("pop_size: must be in 2..4096");
    if (runs < 1) return fail_input("num_runs: must be >= 1");
    if (max_evals < pop) return fail_input("max_evals: must be >= pop_size");
    dock_params p;
    if (params) p = *params; else dock_params_default(&p);
    std::string err;
    if (dk::validate_params(p, &err) != DOCK_OK) return fail_input(err);
    std::vector<float4> packed;
    if (dk::pack_grid(grids, &packed, &err) != DOCK_OK) return fail_input(err);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (n_ligands == 0) return DOCK_OK;

    // ---- devices and slots ----
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        g_screen_error = "no CUDA device (this library has no CPU fallback)";
        return DOCK_E_INTERNAL;
    }
    std::vector<int> devs;
    const int nd = opts && opts->n_devices > 0 ? opts->n_devices : ndev;
    for (int i = 0; i < nd; ++i) {
        const int d = (opts && opts->devices) ? opts->devices[i] : i;
        if (d < 0 || d >= ndev) return fail_input("opts.devices[" + std::to_string(i) + "]: no such CUDA device");
        devs.push_back(d);
    }
    const int slots = opts && opts->slots_per_device > 0 ? std::min(opts->slots_per_device, 64) : 4;
    int prep_threads = opts && opts->prep_threads > 0 ? opts->prep_threads : (int)std::thread::hardware_concurrency();
    prep_threads = std::max(1, std::min(prep_threads, n_ligands));

    // ---- 1. host preprocessing on a thread pool (row a11) ----
    const auto t_prep0 = clk::now();
    std::vector<dk::Prepared> prep(n_ligands);
    std::vector<int> prep_rc(n_ligands, DOCK_OK);
    std::vector<std::string> prep_err(n_ligands);
    {
        std::atomic<int> next{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < prep_threads; ++t)
            pool.emplace_back([&] {
                for (int i; (i = next.fetch_add(1)) < n_ligands;)
                    prep_rc[i] = dk::prepare_ligand(&ligands[i], type_params, grids->n_types, dk::scoring_of(p), &prep[i], &prep_err[i]);
            });
        for (auto &t : pool) t.join();
    }
    const double prep_ms = std::chrono::duration<double, std::milli>(clk::now() - t_prep0).count();

    // ---- 2. LPT order ----
    std::vector<int> order;
    size_t max_blob = 16;
    int n_failed = 0;
    for (int i = 0; i < n_ligands; ++i) {
        if (status) status[i] = prep_rc[i];
        best_energy[i] = NAN;
        if (best_run) best_run[i] = -1;
        if (evals_used) evals_used[i] = 0;
        if (device_of) device_of[i] = -1;
        std::fill(best_genotype + (size_t)i * DOCK_MAX_GENES, best_genotype + (size_t)(i + 1) * DOCK_MAX_GENES, 0.0f);
        if (prep_rc[i] != DOCK_OK) { ++n_failed; continue; }
        order.push_back(i);
        max_blob = std::max(max_blob, prep[i].blob.size());
    }
    auto cost = [&](int i) { return 40.0 * prep[i].P + 133.0 * prep[i].N; };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });

    // ---- 3. receptors and slot contexts ----
    struct Slot { dock_ctx *ctx = nullptr; SlotBufs b; int device = 0; };
    std::vector<Slot> slot_v;
    slot_v.reserve(devs.size() * (size_t)slots);
    int rc = DOCK_OK;
    std::vector<std::shared_ptr<dk::Receptor>> recs;
    auto cleanup = [&] {
        for (auto &s : slot_v) {
            if (s.ctx) { cudaSetDevice(s.device); cudaStreamSynchronize(s.ctx->stream); }
            if (s.ctx) s.b.release(s.ctx->stream);
            dock_free(s.ctx);
        }
        slot_v.clear();
        recs.clear();
    };
    for (int d : devs) {
        std::shared_ptr<dk::Receptor> rec;
        if ((rc = dk::receptor_upload(grids, packed, d, &rec, &err)) != DOCK_OK) { g_screen_error = err; cleanup(); return rc; }
        recs.push_back(rec);
        for (int k = 0; k < slots; ++k) {
            Slot s;
            s.device = d;
            if ((rc = dk::ctx_create(rec, p, &s.ctx, &err)) != DOCK_OK) { g_screen_error = err; cleanup(); return rc; }
            slot_v.push_back(std::move(s));
            Slot &sl = slot_v.back();
            if (!sl.b.h_bE.reserve(runs) || !sl.b.h_bG.reserve((size_t)runs * DOCK_MAX_GENES) || !sl.b.h_ev.reserve(runs)) {
                g_screen_error = "pinned host allocation failed";
                cleanup();
                return DOCK_E_INTERNAL;
            }
            const cudaStream_t st = sl.ctx->stream;
            if ((rc = dk::ctx_reserve(sl.ctx, max_blob, runs, pop)) != DOCK_OK ||
                dk::dmalloc((void **)&sl.b.d_bE, sizeof(float) * runs, st) != cudaSuccess ||
                dk::dmalloc((void **)&sl.b.d_bG, sizeof(float) * runs * DOCK_MAX_GENES, st) != cudaSuccess ||
                dk::dmalloc((void **)&sl.b.d_ev, sizeof(int64_t) * runs, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess) {
                g_screen_error = "slot setup on device " + std::to_string(d) + ": " +
                                 (sl.ctx->err.empty() ? "allocation failed" : sl.ctx->err);
                cudaGetLastError();
                cleanup();
                return DOCK_E_INTERNAL;
            }
        }
    }

    // ---- 4./5. workers ----
    const auto t_dock0 = clk::now();
    std::atomic<size_t> cursor{0};
    std::atomic<bool> abort{false};
    std::atomic<long long> total_evals{0};
    std::mutex err_mu;
    std::string worker_err;
    auto worker = [&](Slot &s) {
        cudaSetDevice(s.device);
        for (size_t k; !abort.load() && (k = cursor.fetch_add(1)) < order.size();) {
            const int i = order[k];
            dock_ctx *c = s.ctx;
            int r = dk::ctx_attach_ligand(c, std::move(prep[i]));
            const uint32_t lid = ligand_ids ? ligand_ids[i] : (uint32_t)i;
            const int G = c->prep.G;
            if (r == DOCK_OK)
                r = dock_run_device(c, pop, runs, 0, lid, max_evals, seed, s.b.d_bE, s.b.d_bG, s.b.d_ev, nullptr,
                                    c->stream);
            if (r == DOCK_OK) {
                cudaError_t e = cudaMemcpyAsync(s.b.h_bE.data(), s.b.d_bE, sizeof(float) * runs, cudaMemcpyDeviceToHost, c->stream);
                if (e == cudaSuccess) e = cudaMemcpyAsync(s.b.h_bG.data(), s.b.d_bG, sizeof(float) * runs * G, cudaMemcpyDeviceToHost, c->stream);
                if (e == cudaSuccess) e = cudaMemcpyAsync(s.b.h_ev.data(), s.b.d_ev, sizeof(int64_t) * runs, cudaMemcpyDeviceToHost, c->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
                if (e != cudaSuccess) { c->err = std::string("result copy: ") + cudaGetErrorString(e); r = DOCK_E_INTERNAL; }
            }
            if (r != DOCK_OK) {
                std::lock_guard<std::mutex> lk(err_mu);
                if (worker_err.empty()) worker_err = "ligand " + std::to_string(i) + " on device " + std::to_string(s.device) + ": " + c->err;
                if (status) status[i] = r;
                abort.store(true);
                return;
            }
            // best over runs: argmin, NaN as +inf, lowest run on ties
            int br = 0;
            float bv = INFINITY;
            long long ev = 0;
            for (int q = 0; q < runs; ++q) {
                const float v = std::isnan(s.b.h_bE[q]) ? INFINITY : s.b.h_bE[q];
                if (v < bv) { bv = v; br = q; }
                ev += s.b.h_ev[q];
            }
            best_energy[i] = s.b.h_bE[br];
            if (best_run) best_run[i] = br;
            std::copy(s.b.h_bG.data() + (size_t)br * G, s.b.h_bG.data() + (size_t)(br + 1) * G,
                      best_genotype + (size_t)i * DOCK_MAX_GENES);
            if (evals_used) evals_used[i] = ev;
            if (device_of) device_of[i] = s.device;
            total_evals.fetch_add(ev);
        }
    };
    {
        std::vector<std::thread> ws;
        for (auto &s : slot_v) ws.emplace_back(worker, std::ref(s));
        for (auto &t : ws) t.join();
    }
    const double dock_ms = std::chrono::duration<double, std::milli>(clk::now() - t_dock0).count();
    long long launches = 0;
    for (auto &s : slot_v) launches += s.ctx->launches;
    cleanup();
    if (stats) {
        stats->prep_ms = prep_ms;
        stats->dock_ms = dock_ms;
        stats->total_evals = total_evals.load();
        stats->n_failed = n_failed;
        stats->launches = launches;
    }
    if (abort.load()) { g_screen_error = worker_err; return DOCK_E_INTERNAL; }
    return DOCK_OK;
}

extern "C" const char *dock_screen_last_error(void) { return g_screen_error.c_str(); }
