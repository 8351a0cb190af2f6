"""Route the reference package's solve path through this GPU implementation.

    import mcstokes.driver
    from paper_2207_08481_b200 import integration
    integration.install(mcstokes.driver)
    mcstokes.driver.run_solve("channel", level, k, nu, opts)   # -> GPU

`install` swaps the reference driver's module-level entry points
(`driver.py:74-180`: `build_system`, `velocity_preconditioner`,
`condensed_rhs`, `solve_stokes`, `post_checks`) for the GPU drop-ins, so the
reference's own callers (`run_solve`, `cli.main`) run the condensation, the
preconditioner and the Krylov solve on the B200.  The GPU `solve_stokes`
reads only `problem.mesh`, `problem.regions`, `problem.body_force` and
`problem.name`, so the reference's `Problem` objects (and their `Mesh` /
`BoundaryRegions`) are accepted as they are.

A finer-grained patch (only `velocity_preconditioner`) would leave the
reference's `cg(lambda v: S_free @ v, ...)` on the host with a host CSR of
S, i.e. the hot path on the CPU; the whole-solve swap keeps it on the GPU.
`uninstall` restores the originals.
"""

from __future__ import annotations

from . import driver as _gpu

_NAMES = ("build_system", "velocity_preconditioner", "condensed_rhs", "solve_stokes",
          "post_checks", "SolverOptions", "SolveResult", "RunRecord")
_SAVED = {}


def install(driver_module):
    """Patch `driver_module` (the reference's `mcstokes.driver`) in place."""
    key = id(driver_module)
    if key not in _SAVED:
        _SAVED[key] = {n: getattr(driver_module, n) for n in _NAMES if hasattr(driver_module, n)}
    for n in _NAMES:
        setattr(driver_module, n, getattr(_gpu, n))
    return driver_module


def uninstall(driver_module):
    """Restore the reference's own entry points."""
    for n, v in _SAVED.pop(id(driver_module), {}).items():
        setattr(driver_module, n, v)
    return driver_module
