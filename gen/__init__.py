"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NONE of the docking method's arithmetic (no pose, no
scoring, no gradient, no search, no pair rule, no RNG of the method).  It only
produces input data: ligands (atoms, charges, coordinates, bonds, rotatable
flags) and receptor grid maps, shaped like the paper's workloads
(§II-A: "21, 43, and 108 atoms, and 2, 15, and 31 rotatable
bonds"; BASELINE.json configs).  The recipe is SURVEY.md §8(d) "Synthetic
inputs" and is restated in DESIGN.md §4.
"""
from .synth import (  # noqa: F401
    TYPE_TABLE, TYPE_NAMES, CONFIGS, make_ligand, make_grid, grid_for_ligand,
    multilinear_grid, planted_grid, constant_grid, config_inputs, hts_ligands,
    random_genotypes,
)
