import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2408_12588_b200.diffusion import Denoiser, initial_latent, make_schedule
from paper_2408_12588_b200.model import ModelConfig, init_model
from paper_2408_12588_b200.policies import PabPolicy, build_schedule
cfg = ModelConfig(layers=2, hidden=144, heads=2, frames=4, spatial_tokens=256, text_tokens=20, cross_in_temporal=True)
params = init_model(cfg, seed=5)
sched = make_schedule(6)
table = build_schedule(PabPolicy(2, 3, 2, window=(990.0, 10.0)), sched, cfg.layers)
den = Denoiser(params, sched, table, np.arange(20), guidance=True, guidance_scale=4.0)
x0 = torch.from_numpy(initial_latent(params, 4, 2)).cuda()
eager = den.run(x0.clone()).cpu()
eager2 = den.run(x0.clone()).cpu()
print("eager repeat equal", torch.equal(eager, eager2))
den.capture_graph()
print("graph launches", den.graph_launches)
g1 = den.run_graph(x0.clone()).cpu()
g2 = den.run_graph(x0.clone()).cpu()
print("graph repeat equal", torch.equal(g1, g2), "graph vs eager equal", torch.equal(g1, eager),
      "rel", float((g1 - eager).norm() / eager.norm()))
