"""In-graph timeline of one draft level (cfg2): stamps around level_inputs / forward / top-k / grow."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_23858_b200 import _lib as L  # noqa: E402

wl = bench.WORKLOADS["cfg2"]
sd, tc, dc = bench.build_decoder(wl, "cfg2", torch.device("cuda"))
sd.prefill(bench.prompts_for(wl, tc.vocab, 0))
sd.step(use_graph=False)
torch.cuda.synchronize()
lib = L.lib()
st = torch.zeros(64, dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
sh = sd.shape
D, W, k = sh.depth, sh.width, sh.expansion_k
dr, g = sd.draft, sd.grown
rows = sd.B * sd.R
idx = [0]


def stamp(sp):
    L.check(lib.ygg_stamp(st.data_ptr() + 8 * idx[0], sp))
    idx[0] += 1


graph = torch.cuda.CUDAGraph()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(graph, stream=s):
    sp = L.stream_ptr(s)
    for _ in range(2):
        stamp(sp)
        L.check(lib.ygg_level_inputs(g.struct, sd.seq.struct, sd.R, k, dr.tokens.data_ptr(), dr.pos.data_ptr(),
                                     dr.slot.data_ptr(), dr.req.data_ptr(), dr.qmask.data_ptr(), dr.mask_words,
                                     dr.blk_start.data_ptr(), dr.blk_len.data_ptr(), sd.cand_n.data_ptr(), sp))
        stamp(sp)
        dr.run(s)
        stamp(sp)
        L.check(lib.ygg_topk_softmax(dr.logits.data_ptr(), L.YGG_F32, rows, dc.vocab, dc.vocab, k, 1.0,
                                     sd.cand_tok.data_ptr(), sd.cand_prob.data_ptr(), None, sd.topk_ws.data_ptr(),
                                     sd.topk_ws.numel(), sp))
        stamp(sp)
        L.check(lib.ygg_egt_grow_level(g.struct, sd.R, k, W, sd.cand_tok.data_ptr(), sd.cand_prob.data_ptr(),
                                       sd.cand_n.data_ptr(), sp))
    stamp(sp)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
t = st.cpu().tolist()[: idx[0]]
d = [(t[i + 1] - t[i]) / 1000 for i in range(len(t) - 1)]
names = ["level_inputs", "forward", "topk", "grow"] * 2
print({n: round(x, 1) for n, x in zip(names[4:], d[4:8])})
