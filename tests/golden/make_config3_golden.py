"""Golden digests of the config-3 growing domain, made by running the
REFERENCE (scantherm 0.1.0) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config3_golden.py

BASELINE configs[3]: 2 x 2 mm footprint on a 2 mm plate, Q1,
MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6), 10 powder
layers.  Per layer: the synthetic state of tests/growth_rule.py,
advance_layer, apply_update, build_dofmap, interface_faces; the sha256
digests of every table (leaf set, numbering, constraints, facets,
transferred T and r_c, transfer report) go to config3_growth.json.
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import scantherm as st  # noqa: E402
from scantherm import interface_faces  # noqa: E402

from growth_rule import layer_record, synthetic_rc, synthetic_T  # noqa: E402


def main():
    mesh = st.MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6)
    geo = st.PartGeometry.chamber((2e-3, 2e-3), 10 * 40e-6, 2e-3, mesh)
    forest = st.build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    T = synthetic_T(0, dofmap.vertices_m())
    dofmap.distribute(T)
    recs = [layer_record(forest, dofmap, interface_faces(forest), T, history.r_c, None)]
    t0 = time.perf_counter()
    for layer in range(geo.n_layers):
        T = synthetic_T(layer, dofmap.vertices_m())
        dofmap.distribute(T)
        rows = forest.active_cells()
        top = (forest.anchor[rows, 2] + forest.size(rows)) * forest.h_fine
        history.r_c[:] = synthetic_rc(layer, history.r_c, top)
        plan = st.advance_layer(forest, history)
        forest, fields, history = st.apply_update(
            forest, plan, [st.NodalField(T, forest.epoch)], history, T_0=303.0)
        dofmap = st.build_dofmap(forest)
        rec = layer_record(forest, dofmap, interface_faces(forest), fields[0].values,
                           history.r_c, plan.transfer_report.vertex_source)
        rec["coarsened_groups"] = len(plan.coarsened_min_rc)
        recs.append(rec)
        print(f"layer {layer}: {rec['n_cells']} leaves, {rec['n_vertices']} vertices, "
              f"{rec['n_slaves']} hanging, {rec['coarsened_groups']} coarsened")
    print(f"reference: {geo.n_layers} layer advances in {time.perf_counter() - t0:.1f} s")
    with open(os.path.join(HERE, "config3_growth.json"), "w") as f:
        json.dump({"layers": recs}, f, indent=0)


if __name__ == "__main__":
    main()
