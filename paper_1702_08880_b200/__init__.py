"""B200-native hot path of the conservative FEM Landau collision operator
(arXiv 1702.08880; reference package `axlandau`).

The O(N^2) FP64 pair integral (per-point friction K and diffusion D) and the
element Jacobian contraction B^T[D,K]B run as hand-written sm_100a CUDA
kernels behind a C ABI (include/landau_b200.h); this package is the thin
Python host side that mirrors the reference's entry points:

    fused_sweep, fused_inner_loop, axisym_tensor_pair   (axlandau.kernel)
    assemble_collision, CollisionMatrix, default_eps_d  (axlandau.assembly)

`install(module)` patches those names into an imported `axlandau` so the
reference's solver / CLI run on the GPU path unchanged.  Multi-GPU outer
point sharding with an NCCL all-gather of the field state lives in
`paper_1702_08880_b200.shard`.
"""

from .assembly import (
    CollisionMatrix,
    assemble_at,
    assemble_collision,
    assemble_species_meshes,
    default_eps_d,
    element_matrices,
    sample_state,
)
from .solver import (CNSolver, StepFailure, backward_euler_step, linear_cn_step, newton_step,
                     species_meshes_step, theta_step)
from .kernel import (
    Accumulators,
    CollisionParams,
    LandauTensorPair,
    QuadPointData,
    axisym_tensor_pair,
    axisym_tensor_pairs,
    coupling,
    elliptic_KE,
    flop_count,
    fused_inner_loop,
    fused_sweep,
)

__version__ = "0.1.0"

_PATCH = {
    "kernel": ("fused_sweep", "fused_inner_loop"),
    "assembly": ("fused_sweep", "assemble_collision"),
    "solver": ("assemble_collision", "_assemble_at", "newton_step", "linear_cn_step"),
    "cli": ("assemble_collision", "fused_sweep"),
}


def _assemble_at_cfg(mesh, ref, state, params, cfg):
    """solver._assemble_at signature (solver.py:81-84): device sampling +
    operator in one call."""
    return assemble_at(mesh, ref, state, params, eps_d=getattr(cfg, "eps_d", None))


def install(axlandau_pkg) -> dict:
    """Route an imported reference package through the B200 path.

    The reference imports these names by value (assembly.py:38-43,
    solver.py:32, cli.py:27-29), so every importing module's attribute is
    replaced.  Returns the originals so callers can restore them.
    """
    import importlib

    from . import solver as _solver

    here = {"fused_sweep": fused_sweep, "fused_inner_loop": fused_inner_loop,
            "assemble_collision": assemble_collision, "_assemble_at": _assemble_at_cfg,
            "newton_step": _solver.newton_step, "linear_cn_step": _solver.linear_cn_step}
    saved = {}
    ref_solver = importlib.import_module(f"{axlandau_pkg.__name__}.solver")
    if hasattr(ref_solver, "StepFailure"):  # so the reference's advance() catches ours
        saved[("@", "StepFailure")] = _solver._StepFailure
        _solver._StepFailure = ref_solver.StepFailure
    for mod_name, names in _PATCH.items():
        mod = importlib.import_module(f"{axlandau_pkg.__name__}.{mod_name}")
        for nm in names:
            if hasattr(mod, nm):
                saved[(mod_name, nm)] = getattr(mod, nm)
                setattr(mod, nm, here[nm])
    for nm in ("fused_sweep", "fused_inner_loop", "assemble_collision"):
        if hasattr(axlandau_pkg, nm):
            saved[("", nm)] = getattr(axlandau_pkg, nm)
            setattr(axlandau_pkg, nm, here[nm])
    return saved


def uninstall(axlandau_pkg, saved: dict) -> None:
    import importlib

    for (mod_name, nm), fn in saved.items():
        if mod_name == "@":  # our solver's failure class
            from . import solver as _solver

            _solver._StepFailure = fn
            continue
        mod = axlandau_pkg if not mod_name else importlib.import_module(
            f"{axlandau_pkg.__name__}.{mod_name}")
        setattr(mod, nm, fn)


__all__ = [
    "Accumulators", "CollisionMatrix", "CollisionParams", "LandauTensorPair",
    "QuadPointData", "assemble_at", "assemble_collision", "assemble_species_meshes", "sample_state", "axisym_tensor_pair", "axisym_tensor_pairs",
    "coupling", "default_eps_d", "element_matrices", "elliptic_KE", "flop_count", "fused_inner_loop",
    "fused_sweep", "install", "uninstall", "CNSolver", "StepFailure", "linear_cn_step",
    "backward_euler_step", "theta_step", "species_meshes_step",
    "newton_step",
]
