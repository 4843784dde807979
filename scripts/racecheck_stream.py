"""compute-sanitizer --tool racecheck target: the streamed local kernel alone (hex p = 3 Poisson, 8 elements), with the
stage copies whole (local_ed_stream = 3) or split into 4-row pieces (7)."""
import sys
sys.path.insert(0, '/root/repo')
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
hdg.set_tuning("local_ed_stream", int(sys.argv[1]) if len(sys.argv) > 1 else 3)
disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=3)
model = hdg.make_case_model(disc, "poisson")
ops = hdg.assemble_element_operators(disc, model, hdg.make_initial_state(disc, model))
print("ok")
ctx.close()
