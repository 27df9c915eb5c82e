// prep.h — host-side preprocessing of a ligand and a receptor grid (row a11).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dock.h"
#include "dock_internal.h"

namespace dk {

struct Prepared {
    int N = 0, T = 0, G = 0, P = 0;
    // D1 results in caller atom order
    std::vector<int> tor_a, tor_b, tor_depth;     // [T], torsion order (depth, a, b)
    std::vector<uint8_t> moved;                   // [T*N]
    std::vector<int> pairs;                       // [P*2] lexicographic, i < j
    // device numbering
    std::vector<int> dfs2orig, orig2dfs;          // [N]
    LigDev layout;                                // offsets + sizes (blob pointer unset)
    std::vector<uint8_t> blob;                    // the constant block, layout.blob_bytes
};

// Scoring function of a context (dock_params.scoring and the D5-AD4 coefficients, NEXT-2).
struct Scoring {
    int sf = 0;                   // DOCK_SF_D5 or DOCK_SF_AD4
    double w_vdw = 1, w_hb = 1, w_el = 1, w_ds = 1, w_tors = 0, qasp = 0;
};
Scoring scoring_of(const dock_params &p);

// D1 + blob assembly (pair constants in the form of `sf`).  Returns DOCK_OK or
// DOCK_E_INPUT with `err` naming the field/index.
int prepare_ligand(const dock_ligand *l, const dock_type_param *tp, int n_types, const Scoring &sf, Prepared *out,
                   std::string *err);

// The per-type parameters of a grid (DESIGN.md §3 D5): `tp` if given, else the built-in
// table by grids->type_names (dock_builtin_type_param).  Also validates type_names when
// present (NUL-terminated within 4 chars, non-empty, unique).  DOCK_OK or DOCK_E_INPUT.
int resolve_type_params(const dock_grids *g, const dock_type_param *tp, std::vector<dock_type_param> *out,
                        std::string *err);

// Grid validation and packing into one float4 {M_type, M_E, M_D, 0} per (type, node).
int pack_grid(const dock_grids *g, std::vector<float4> *packed, std::string *err);

}  // namespace dk
