"""Diagnostic: how often would the fused merge flag half-tiles on the bench model's
first decoder step?  (partial = 64 tokens of a 192-token tile)"""
import numpy as np
import paper_1804_05038_b200 as pb

DIMS = dict(src_vocab=32000, tgt_vocab=50000, embed=512, hidden=1024, attn=2048, readout=512)
params = pb.synthetic_model(pb.Dims(**DIMS), 1804)
qm = pb.quantize_model(params)
net = pb.build_network(qm)
rng = np.random.default_rng(0)
flags, rows, fulls = [], 0, 0
for it in range(16):
    src = rng.integers(3, 32000, int(rng.integers(5, 100)))
    enc = net.encode(src)
    lp, st, _ = net.decoder_step(np.array([2]), net.initial_state(enc, 1), enc)
    x = lp[:, 0].astype(np.float64)          # log-probs: same order as logits
    V = x.shape[0]
    nb = (V + 191) // 192
    part_max, part_2nd = [], []
    for b in range(nb * 3):
        t0 = (b // 3) * 192 + (b % 3) * 64
        seg = x[t0:min(t0 + 64, V)]
        if len(seg) == 0:
            continue
        s = np.sort(seg)[::-1]
        part_max.append(s[0]); part_2nd.append(s[1] if len(s) > 1 else -np.inf)
    pm = np.array(part_max); p2 = np.array(part_2nd)
    thr = np.sort(pm)[::-1][7]
    nf = int((p2 >= thr).sum())
    flags.append(nf)
    top = np.sort(x)[::-1][:10]
    print(it, "flagged", nf, "top10 lp", np.round(top, 7).tolist(), "distinct top10", len(set(top.tolist())))
print("mean flagged", np.mean(flags))
