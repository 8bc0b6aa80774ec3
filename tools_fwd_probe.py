# scratch probe: time fold_forward per kernel class on C2 B=1024
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, foldgen
from paper_1702_02181_b200 import fold
gr = foldgen.config_c2(1024); S = 1024
p = foldgen.make_params("treelstm", S, gr.vocab)
dev = "cuda"
model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev))
op, child, token, root = fold.graphs_to_device(gr)
s = fold.schedule(op, child, token, root, gr.vocab)
ws = fold.Workspace(dev)
for _ in range(3): fold.forward(s, model, ws=ws)
torch.cuda.synchronize()
fold.profile_enable(True)
for _ in range(5): fold.forward(s, model, ws=ws)
torch.cuda.synchronize()
pr = fold.profile_read()
print(os.environ.get("FOLD_DBG_FWD_EPI"), {k: round(v[0] / 5, 3) for k, v in pr.items() if v[1]})
