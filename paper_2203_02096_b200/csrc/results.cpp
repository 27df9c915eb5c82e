// results.cpp — NEXT-3: serialisation of a docking result (DESIGN.md
// §12).  The paper removed file writing to time the kernels; a usable docking
// tool needs it back, outside the timed path.  JSON and CSV, floats as %.9g (float32
// round-trips exactly), NaN as JSON null / empty CSV field.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dock.h"

namespace {

void put_f(std::string &o, float v, bool json) {
    if (std::isnan(v) || std::isinf(v)) {
        if (json) o += "null";
        return;
    }
    char b[32];
    std::snprintf(b, sizeof b, "%.9g", (double)v);
    o += b;
}

void put_d(std::string &o, double v) {
    char b[40];
    if (std::isnan(v) || std::isinf(v)) { o += "null"; return; }
    std::snprintf(b, sizeof b, "%.17g", v);
    o += b;
}

void put_i(std::string &o, long long v) { o += std::to_string(v); }

void put_s(std::string &o, const char *s) {
    o += '"';
    for (const char *p = s ? s : ""; *p; ++p) {
        const unsigned char ch = (unsigned char)*p;
        if (ch == '"' || ch == '\\') { o += '\\'; o += (char)ch; }
        else if (ch < 0x20) { char b[8]; std::snprintf(b, sizeof b, "\\u%04x", ch); o += b; }
        else o += (char)ch;
    }
    o += '"';
}

float key(float e) { return std::isnan(e) ? INFINITY : e; }

}  // namespace

extern "C" int dock_write_result(const dock_result_view *r, int32_t format, char *buf, size_t cap, size_t *len) {
    if (!r || (format != DOCK_FMT_JSON && format != DOCK_FMT_CSV)) return DOCK_E_INPUT;
    if (r->n_runs < 0 || r->n_atoms < 0 || r->n_genes < 0 || r->n_timings < 0) return DOCK_E_INPUT;
    if (r->n_runs > 0 && !r->best_energy) return DOCK_E_INPUT;
    if (r->n_runs > 0 && r->n_genes > 0 && !r->best_genotype) return DOCK_E_INPUT;
    if (r->n_timings > 0 && (!r->timing_names || !r->timing_ms)) return DOCK_E_INPUT;
    const int R = r->n_runs, G = r->n_genes, N = r->n_atoms;
    // best = minimum over runs, NaN as +inf, lowest run on ties
    int best = -1;
    for (int i = 0; i < R; ++i)
        if (best < 0 || key(r->best_energy[i]) < key(r->best_energy[best])) best = i;
    std::string o;
    if (format == DOCK_FMT_CSV) {
        o += "run,best_energy,evals,generations,cluster,rmsd_to_seed,dG\n";
        for (int i = 0; i < R; ++i) {
            put_i(o, i); o += ',';
            put_f(o, r->best_energy[i], false); o += ',';
            if (r->evals) put_i(o, r->evals[i]);
            o += ',';
            if (r->generations) put_i(o, r->generations[i]);
            o += ',';
            if (r->cluster) put_i(o, r->cluster[i]);
            o += ',';
            if (r->rmsd_to_seed) put_f(o, r->rmsd_to_seed[i], false);
            o += ',';
            if (r->dG) put_f(o, r->dG[i], false);
            o += '\n';
        }
    } else {
        o += "{\"best_energy\": ";
        if (best >= 0) put_f(o, r->best_energy[best], true); else o += "null";
        o += ", \"best_run\": ";
        put_i(o, best);
        o += ", \"best_genotype\": [";
        for (int j = 0; best >= 0 && j < G; ++j) { if (j) o += ", "; put_f(o, r->best_genotype[(size_t)best * G + j], true); }
        o += "], \"best_coordinates\": [";
        if (best >= 0 && r->best_xyz)
            for (int a = 0; a < N; ++a) {
                if (a) o += ", ";
                o += '[';
                for (int d = 0; d < 3; ++d) { if (d) o += ", "; put_f(o, r->best_xyz[((size_t)best * N + a) * 3 + d], true); }
                o += ']';
            }
        o += "], \"per_run\": [";
        for (int i = 0; i < R; ++i) {
            if (i) o += ", ";
            o += "{\"run\": "; put_i(o, i);
            o += ", \"best_energy\": "; put_f(o, r->best_energy[i], true);
            if (r->evals) { o += ", \"evals\": "; put_i(o, r->evals[i]); }
            if (r->generations) { o += ", \"generations\": "; put_i(o, r->generations[i]); }
            if (r->cluster) { o += ", \"cluster\": "; put_i(o, r->cluster[i]); }
            if (r->rmsd_to_seed) { o += ", \"rmsd_to_seed\": "; put_f(o, r->rmsd_to_seed[i], true); }
            if (r->dG) { o += ", \"dG\": "; put_f(o, r->dG[i], true); }
            o += '}';
        }
        o += "], \"clusters\": [";
        if (r->cluster) {
            int nc = 0;
            for (int i = 0; i < R; ++i) nc = std::max(nc, r->cluster[i] + 1);
            std::vector<int> size(nc, 0), bestc(nc, -1);
            for (int i = 0; i < R; ++i) {
                const int c = r->cluster[i];
                if (c < 0) continue;
                ++size[c];
                if (bestc[c] < 0 || key(r->best_energy[i]) < key(r->best_energy[bestc[c]])) bestc[c] = i;
            }
            for (int c = 0; c < nc; ++c) {
                if (c) o += ", ";
                o += "{\"id\": "; put_i(o, c);
                o += ", \"size\": "; put_i(o, size[c]);
                o += ", \"best_run\": "; put_i(o, bestc[c]);
                o += ", \"best_energy\": ";
                if (bestc[c] >= 0) put_f(o, r->best_energy[bestc[c]], true); else o += "null";
                o += '}';
            }
        }
        o += "], \"timings\": {";
        for (int t = 0; t < r->n_timings; ++t) {
            if (t) o += ", ";
            put_s(o, r->timing_names[t]);
            o += ": ";
            put_d(o, r->timing_ms[t]);
        }
        o += "}}\n";
    }
    if (len) *len = o.size() + 1;
    if (!buf || cap < o.size() + 1) return DOCK_E_INPUT;
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return DOCK_OK;
}

extern "C" int dock_write_screen(int32_t n, const uint32_t *ids, const float *best_energy, const int32_t *best_run,
                                 const float *best_genotype, const int32_t *n_genes, const int64_t *evals,
                                 const int32_t *status, const int32_t *device_of, int32_t format, char *buf,
                                 size_t cap, size_t *len) {
    if (n < 0 || (n > 0 && !best_energy) || (format != DOCK_FMT_JSON && format != DOCK_FMT_CSV)) return DOCK_E_INPUT;
    auto ok = [&](int i) { return !status || status[i] == DOCK_OK; };
    int best = -1;
    for (int i = 0; i < n; ++i)
        if (ok(i) && (best < 0 || key(best_energy[i]) < key(best_energy[best]))) best = i;
    std::string o;
    if (format == DOCK_FMT_CSV) {
        o += "ligand,id,status,best_energy,best_run,evals,device\n";
        for (int i = 0; i < n; ++i) {
            put_i(o, i); o += ',';
            put_i(o, ids ? (long long)ids[i] : i); o += ',';
            put_i(o, status ? status[i] : 0); o += ',';
            put_f(o, best_energy[i], false); o += ',';
            if (best_run) put_i(o, best_run[i]);
            o += ',';
            if (evals) put_i(o, evals[i]);
            o += ',';
            if (device_of) put_i(o, device_of[i]);
            o += '\n';
        }
    } else {
        o += "{\"ligands\": [";
        for (int i = 0; i < n; ++i) {
            if (i) o += ", ";
            o += "{\"ligand\": "; put_i(o, i);
            o += ", \"id\": "; put_i(o, ids ? (long long)ids[i] : i);
            o += ", \"status\": "; put_i(o, status ? status[i] : 0);
            o += ", \"best_energy\": "; put_f(o, best_energy[i], true);
            if (best_run) { o += ", \"best_run\": "; put_i(o, best_run[i]); }
            if (evals) { o += ", \"evals\": "; put_i(o, evals[i]); }
            if (device_of) { o += ", \"device\": "; put_i(o, device_of[i]); }
            if (best_genotype && n_genes && ok(i)) {
                o += ", \"best_genotype\": [";
                for (int j = 0; j < n_genes[i] && j < DOCK_MAX_GENES; ++j) {
                    if (j) o += ", ";
                    put_f(o, best_genotype[(size_t)i * DOCK_MAX_GENES + j], true);
                }
                o += ']';
            }
            o += '}';
        }
        o += "], \"best\": {\"ligand\": "; put_i(o, best);
        o += ", \"best_energy\": ";
        if (best >= 0) put_f(o, best_energy[best], true); else o += "null";
        o += "}}\n";
    }
    if (len) *len = o.size() + 1;
    if (!buf || cap < o.size() + 1) return DOCK_E_INPUT;
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return DOCK_OK;
}
