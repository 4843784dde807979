import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2512_13619_b200 as hdg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3, jitter=0.1)
model = hdg.make_case_model(disc, "poisson")
state = hdg.make_initial_state(disc, model)
rng = np.random.default_rng(1)
state.u = state.u + 0.1 * rng.standard_normal(state.u.shape)
state.uhat = state.uhat + 0.1 * rng.standard_normal(state.uhat.shape)
names = ["kbar", "e_raw", "d_raw0", "d_raw1", "d_raw2", "h_raw", "g_raw0", "g_raw1", "g_raw2", "f_raw", "j_raw"]
for mode in (3,):
    hdg.set_tuning("local_ed_stream", mode)
    ref = {}
    for r in range(R):
        ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
        for nm in names:
            a = ops.get(nm)
            if r == 0:
                ref[nm] = a
            elif not np.array_equal(a, ref[nm]):
                a2 = a.reshape(disc.ne, -1) if a.size % disc.ne == 0 else a
                r2 = ref[nm].reshape(a2.shape)
                bad = np.argwhere(a2 != r2)
                els = np.unique(bad[:, 0])
                print("mode", mode, "run", r, nm, "differs:", len(bad), "entries in", len(els), "elements", els[:8],
                      "rows", sorted(set((bad[:, 1] % 64).tolist())) if nm[0] in "ed" else None, "cols", sorted(set((bad[:, 1] // 64).tolist())) if nm[0] in "ed" else None, "max abs", np.abs(a2 - r2).max(), "vals", a2[bad[0, 0], bad[0, 1]], r2[bad[0, 0], bad[0, 1]])
        del ops
    print("mode", mode, "done")
ctx.close()
