// engine.h — host-side engine objects shared by the single-ligand ABI (dock_abi.cpp)
// and the multi-ligand / multi-GPU scheduler (screen.cpp).
//
//   Receptor  one upload of the packed grid maps per device ("every GPU
//             holds its own copy of the receptor grid"); shared by every context on it.
//   dock_ctx  one (device, stream, ligand block, population buffers) engine.  A screen
//             worker keeps one dock_ctx per in-flight slot and swaps ligands into it.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/dock.h"
#include "kernels.cuh"
#include "prep.h"

namespace dk {

// Stream-ordered device memory (cudaMallocAsync / cudaFreeAsync from the device's default
// pool, release threshold raised so freed blocks stay cached in the process).  A plain
// cudaFree synchronises the device and was measured at 100-400 ms per context teardown
// on B200 (profiles/r01f, DOCK_TRACE); pool frees are asynchronous and cheap.
void pool_setup(int device);
inline cudaError_t dmalloc(void **p, size_t bytes, cudaStream_t s) { return cudaMallocAsync(p, bytes ? bytes : 16, s); }
inline void dfree(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Pinned host blocks for the small per-batch device->host reads (termination poll, screen
// results), cached for the life of the process: cudaFreeHost is slow, and pageable
// copies from several worker threads serialise through the driver's staging buffer
// (measured: dock_screen with 4 slots lost 25 % with pageable polls, profiles/r01o).
void *pinned_get(size_t bytes);
void pinned_put(void *p, size_t bytes);
template <typename T>
struct PinnedBuf {
    T *p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf &) = delete;
    PinnedBuf &operator=(const PinnedBuf &) = delete;
    PinnedBuf(PinnedBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    ~PinnedBuf() { if (p) pinned_put(p, n * sizeof(T)); }
    bool reserve(size_t count) {
        if (count <= n) return true;
        if (p) pinned_put(p, n * sizeof(T));
        p = static_cast<T *>(pinned_get(count * sizeof(T)));
        n = p ? count : 0;
        return p != nullptr;
    }
    T &operator[](size_t i) { return p[i]; }
    T *data() { return p; }
};

struct Receptor {
    int device = 0;
    cudaStream_t stream = nullptr;   // owns the upload and the final free
    float4 *d_maps = nullptr;
    size_t bytes = 0;
    GridDev grid{};
    Receptor() = default;
    Receptor(const Receptor &) = delete;
    Receptor &operator=(const Receptor &) = delete;
    ~Receptor();
};

// Upload packed maps (pack_grid output) to `device`.  DOCK_OK / DOCK_E_INTERNAL.
int receptor_upload(const dock_grids *g, const std::vector<float4> &packed, int device,
                    std::shared_ptr<Receptor> *out, std::string *err);

}  // namespace dk

struct dock_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::shared_ptr<dk::Receptor> rec;
    dk::Prepared prep;
    dk::LigDev lig{};
    dk::GridDev grid{};
    dock_params params{};
    uint8_t *d_blob = nullptr;
    size_t blob_cap = 0;
    int *d_dfs2orig = nullptr;
    int cap_runs = 0, cap_pop = 0;
    float *d_genes = nullptr, *d_E = nullptr;
    dk::RunState *d_state = nullptr;
    int *d_perm = nullptr, *d_ls_evals = nullptr, *d_ls_count = nullptr;
    unsigned *d_spec_done = nullptr;            // k_run_sw speculative GA bitmaps [runs][2][ceil(pop/32)]
    int *d_spec_ctr = nullptr;                  // [runs][2]
    dk::PinnedBuf<dk::RunState> h_state;   // termination poll target
    std::string err;
    long long launches = 0;
    double prof_ms[3] = {0, 0, 0};
    long long prof_n[3] = {0, 0, 0};
    std::vector<cudaEvent_t> events;   // profiling: 3 per captured generation + 2 for init
    std::vector<cudaStream_t> branch_streams;   // run branches of the generation graph (run_branches)
    std::vector<cudaEvent_t> branch_events;     // fork + one join per branch (timing disabled)
    int last_branches = 1;
    int last_engine = 0;        // dock_last_engine: 0 lockstep, 1 run branches, 2 persistent clusters
    unsigned long long *d_prof = nullptr;       // k_run_sw LS-phase timer (profile)
    // Recorded after the last kernel of every device-side call (dock_run_device and the
    // stream-taking hooks may return before their kernels finish).  Every later use of the
    // context's buffers -- a reallocation, a ligand swap, dock_free, a hook on c->stream,
    // another dock_run_device on any stream -- is ordered after it (dk::after_last_use).
    cudaEvent_t last_use = nullptr;
};

namespace dk {

// New context on rec->device with its own non-blocking stream and the grid's L2
// persistence window (NS).  No ligand attached yet.
int ctx_create(std::shared_ptr<Receptor> rec, const dock_params &p, dock_ctx **out, std::string *err);

// Move a prepared ligand into the context and upload its constant block on the context's
// stream.  Device buffers only grow (reserve_blob pre-sizes them so a screen never frees
// device memory, which would synchronise the whole device, while other slots run).
int ctx_attach_ligand(dock_ctx *c, Prepared &&p);
int ctx_reserve(dock_ctx *c, size_t blob_bytes, int runs, int pop);

int validate_params(const dock_params &p, std::string *err);

// Order stream s after the context's last recorded device-side use (cudaStreamWaitEvent),
// and record a new last use at the current end of s.
cudaError_t after_last_use(dock_ctx *c, cudaStream_t s);
cudaError_t mark_last_use(dock_ctx *c, cudaStream_t s);

}  // namespace dk
