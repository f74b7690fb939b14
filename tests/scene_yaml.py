"""Scenario YAML templates for BASELINE configs 2/3/5 (SURVEY.md §8d and
Appendix C), through the reference's own scenario schema (harness.py
parse_scenario). No imports of the product or the reference, so the golden
generator (which runs the REFERENCE) and the tests share one template."""

from __future__ import annotations


def block_yaml(cx, cy, cz, frac, h=0.05, frames=20, collider="plane", outer=1, inner=1, vel=-0.01):
    """SURVEY Appendix C block template (configs 2/3/5). collider 'plane' =
    half-space sinking 1 cm/frame; 'jaw' = capsule on a rotate motion
    (articulated self-contact emulation)."""
    ex, ey, ez = cx * h, cy * h, cz * h
    if collider == "plane":
        cold = (f"  - shape: {{half_space: {{point: [0.0, 0.0, {ez + 0.01}], normal: [0.0, 0.0, -1.0]}}}}\n"
                f"    motion: {{kind: translate, velocity: [0.0, 0.0, {vel}]}}\n")
    else:
        r = 0.3 * ey
        cold = (f"  - shape: {{capsule: {{p0: [{0.2 * ex}, -0.2, {ez + r - 0.02}], p1: [{0.2 * ex}, {ey + 0.2}, "
                f"{ez + r - 0.02}], radius: {r}}}}}\n"
                f"    motion: {{kind: rotate, axis_point: [0.0, {ey / 2}, {ez + r}], axis_dir: [0.0, 1.0, 0.0], "
                f"degrees_per_frame: 1.0}}\n")
    return f"""
name: block_{cx}_{cy}_{cz}
mesh: {{lattice: {{extent: [{ex}, {ey}, {ez}], cells: [{cx}, {cy}, {cz}]}}}}
material: {{mu: 1.0e+4}}
attachments:
  - name: base
    region: {{box: {{min: [-0.1, -0.1, -0.1], max: [{ex + 0.1}, {ey + 0.1}, {h / 2}]}}}}
    stiffness: 1.0e+7
    motion: {{kind: fixed}}
proxies:
  region: {{box: {{min: [-0.1, -0.1, {ez - h / 2}], max: [{frac * ex + 1e-6}, {ey + 0.1}, {ez + 0.1}]}}}}
colliders:
{cold}solver: {{kind: schur, outer_iters: {outer}, inner_iters: {inner}}}
frames: {frames}
"""


CONFIGS = {
    "cfg1": None,  # tests/golden/cfg1.npz yaml (beam 20x8x8, 5 % prone)
    "cfg2": (40, 25, 20, 0.7),
    "cfg3": (80, 50, 30, 1.0),
    "cfg5": (50, 30, 20, 0.75),
}
