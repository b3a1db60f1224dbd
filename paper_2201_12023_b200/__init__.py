"""B200-native executor for Alpa plans (arXiv 2201.12023).

Plans come unchanged from the reference planner (`meshplan`, plan.json); this
package executes them on sm_100a GPUs: per-stage SPMD sharded operators on
hand-written tcgen05/TMA kernels (libmpexec.so, C-ABI in include/mp_exec.h),
intra-mesh collectives and cross-mesh resharding over NCCL, and a GPipe/1F1B
microbatch runtime.  The public entry point is `execute` (runtime.py), the
drop-in for the reference's `emit_instructions -> simulate` path.
"""
__version__ = "0.1.0"
