"""Render profiles/<tag>_configs.json (tools/bench_configs.py) as markdown."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
d = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_configs.json")))
c1, c2, c3, c4, c5 = (d[k] for k in ("C1", "C2", "C3", "C4", "C5"))
L = [f"# {tag}: per-config evidence (BASELINE.json configs C1-C5), one B200, FP64 unless stated\n",
     f"Produced by `python tools/bench_configs.py {tag}` on the GPU box and rendered by "
     f"`tools/configs_md.py`. The raw numbers are in\n`{tag}_configs.json`. The reference "
     "(`oracle/_ref`, compiled from its own sources) was timed\non the same box's host cores "
     f"({d['cores']} threads available).\n",
     "## C1: 256x64 D2Q9+D2Q9 BGK, primal to steady state, then adjoint and gradient\n",
     "**Protocol (c): GPU-only convergence.** The geometry is SURVEY A.3 (initial_w 0.5, no noise).\n",
     "| iteration | GPU exact objective | reference trace (SURVEY A.3) | abs diff |\n|---|---|---|---|"]
for k, v in c1["trace_exact"].items():
    L.append(f"| {int(k):,} | {v['objective']:.16g} | {v['reference_trace']:.16g} | {v['abs_diff']:.1e} |")
n0, e0 = c1["noise0_fast"], c1["noise0_exact"]
L.append(f"\nConvergence to tol 1e-10:\n- product build: {n0['primal_iterations']:,} iterations in "
         f"{n0['seconds']:.2f} s ({n0['steps_per_s']:,.0f} steps/s), objective {n0['objective']:.16g};\n"
         f"- exact build: {e0['primal_iterations']:,} iterations in {e0['seconds']:.2f} s, objective "
         f"{e0['objective']:.16g}.\n")
L.append("SURVEY's value of 0.01066509204221 was read off the trace at ≤400K iterations (residual "
         "3.7e-8). The slow\nthermal mode still moves the objective by 1.6e-10 between there and "
         "tol 1e-10. The exact build\nreproduces the reference's own trace to ≤4e-17 at 25K, 100K "
         "and 400K iterations, so 0.0106650918798\nis the reference's converged value too.\n")
fp = c1["fixed_iteration_parity"]
L.append(f"**Protocol (a): fixed-iteration parity.** {fp['steps']:,} primal steps, then {fp['steps']:,} "
         "adjoint sweeps, exact build against\nthe reference itself:\n"
         f"- state equal: {fp['state_equal']};\n- adjoint equal: {fp['adjoint_equal']};\n"
         f"- objective equal: {fp['objective_equal']};\n"
         f"- gradient + inlet_dp equal: {fp['gradient_equal']} (bitwise).\n\n"
         f"The reference runs {fp['reference_primal_steps_per_s_1thread']:.0f} steps/s on 1 thread, "
         f"so the C1 primal solve would take ≈{fp['reference_seconds_for_case_primal_solve_est']/60:.0f} "
         "min on the CPU.\n")
cs = c1["case"]
L.append(f"**The C1 case itself** (noise 0.3, seed 7):\n- primal: {cs['primal_iterations']:,} "
         f"iterations to 1e-10 in {cs['primal_seconds']:.1f} s;\n- adjoint: "
         f"{cs['adjoint_iterations']:,} sweeps, residual {cs['adjoint_residual']:.2e}, converged "
         f"{cs['adjoint_converged']} (max_inner 3M is the config's cap);\n- adjoint + gradient: "
         f"{cs['adjoint_plus_gradient_seconds']:.1f} s.\n")
L.append("## C2: 1024x256 mixer, warm start, then 50 one-shot iterations at zeta 1e-4\n")
L.append(f"- GPU (product build): {c2['gpu_iterations_per_s']:,.0f} iterations/s. The reference on "
         f"1 thread: {c2['reference_iterations_per_s']:.2f} iterations/s "
         f"({c2['gpu_iterations_per_s']/c2['reference_iterations_per_s']:,.0f}x).\n"
         f"- On the same warm (f, v, w), after 50 iterations:\n"
         f"  - max |w_gpu - w_ref| = {c2['max_abs_w_diff']:.1e};\n"
         f"  - objective trace max relative diff {c2['max_rel_objective_diff']:.1e};\n"
         f"  - gradient-norm trace {c2['max_rel_gradnorm_diff']:.1e}.\n"
         f"- The design moved by {c2['design_moved']:.1e}.\n")
L.append("## C3: 256x128x128 mixer3d (D3Q19+D3Q7), sweep rates\n")
L.append("| variant | primal MLUPS (GB/s) | adjoint MLUPS (GB/s) | pair MLUPS (`lbgpu_pair_steps`) | "
         "frozen-base adjoint MLUPS |\n|---|---|---|---|---|")
for k, v in c3.items():
    L.append(f"| {k} | {v['primal_mlups']:,.0f} ({v['primal_gbs']:,.0f}) | {v['adjoint_mlups']:,.0f} "
             f"({v['adjoint_gbs']:,.0f}) | {v.get('pair_mlups', float('nan')):,.0f} | "
             f"{v.get('adjoint_frozen_base_mlups', float('nan')):,.0f} |")
_pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6529.4
L.append(f"\nMeasured copy peak: {_pk:,.1f} GB/s. The pair is fused (one k_pair sweep) at FP64 and runs "
         "apart at FP32.\n")
L.append("## C4: 512x128x128 exchanger3d topology optimisation\n")
for key, title in (("parity_128x32x32", "128x32x32 (C4 proportions)"),
                   ("parity_full_size", "full size 512x128x128")):
    p = c4.get(key)
    if p:
        L.append(f"**Parity at {title}.** {p['warm_iterations']} zeta = 0 warm-up iterations on the "
                 f"GPU, then {p['iterations']} one-shot iterations at zeta 1e-4 on both engines from the "
                 f"same (f, v, w):\n- max |w_gpu - w_ref| = {p['max_abs_w_diff']:.1e};\n"
                 f"- objective trace {p['max_rel_objective_diff']:.1e} relative;\n"
                 f"- gradient-norm trace {p['max_rel_gradnorm_diff']:.1e};\n"
                 f"- design moved {p['design_moved']:.1e};\n"
                 f"- reference {p['reference_seconds_1thread']:.1f} s on 1 thread.\n")
L.append(f"**Throughput.**\n- One-shot: {c4['one_shot_iterations_per_s']:.0f} iterations/s, i.e. "
         f"{c4['one_shot_node_iterations_mlups']:,.0f} M node-iterations/s. Each iteration is "
         "primal + adjoint + gradient/update; the update of a non-record iteration rides in the "
         "next iteration's primal sweep (k_primal UPD).\n"
         f"- Sweeps: primal {c4['primal_gbs']:,.0f} GB/s, adjoint {c4['adjoint_gbs']:,.0f} GB/s.\n"
         f"- The reference on {c4['reference_cores']} threads: "
         f"{c4['reference_primal_plus_adjoint_seconds_per_iteration']:.2f} s per primal+adjoint "
         f"iteration, against {1/c4['one_shot_iterations_per_s']*1e3:.2f} ms here.\n")
L.append("## C5: 2048x512x512 over 8 GPUs, one rank's slab on one GPU\n")
L.append(f"- Slab 0 of 8 (256 owned columns + ghosts, {c5['owned_nodes']:,} nodes): primal "
         f"{c5['primal_mlups']:,.0f} MLUPS ({c5['primal_gbs']:,.0f} GB/s), adjoint "
         f"{c5['adjoint_mlups']:,.0f} MLUPS ({c5['adjoint_gbs']:,.0f} GB/s), over owned nodes.\n"
         "- Unsteady adjoint on a standalone 256x512x512 lattice with the C5 physics (one rank's "
         "node count):\n"
         f"  - {c5['unsteady_warmup_steps']} warm-up steps, then N_t = {c5['unsteady_steps']};\n")
if "unsteady_by_slots" in c5:
    L.append(f"  - round 1 (recursive bisection, 4 slots): "
             f"{c5['unsteady_round1_forward_sweeps_4_slots']:,} primal sweeps;\n")
    for k, u in c5["unsteady_by_slots"].items():
        L.append(f"  - binomial schedule, {k} slots: {u['forward_sweeps']:,} primal sweeps "
                 f"({u['recompute_factor']:.2f} N_t) and {u['adjoint_sweeps']} adjoint sweeps in "
                 f"{u['seconds']:.1f} s, {u['node_sweeps_per_s_mlups']:,.0f} M node-sweeps/s; "
                 f"J = {u['J']:.6g}, max |dJ/dw| = {u['grad_max']:.3e}.\n")
else:
    L.append(f"  - {c5['unsteady_slots']} checkpoint slots: {c5['unsteady_forward_sweeps']:,} primal "
             f"sweeps and {c5['unsteady_adjoint_sweeps']} adjoint sweeps in "
             f"{c5['unsteady_seconds']:.1f} s; J = {c5['unsteady_J']:.6g}.\n")
open(os.path.join(ROOT, "profiles", f"{tag}_configs.md"), "w").write("\n".join(L) + "\n")
print("ok")
