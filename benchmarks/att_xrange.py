import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1804_05038_b200 as pb
d = pb.Dims(32000, 50000, 512, 1024, 2048, 512)
params = pb.synthetic_model(d, 1804)
qm = pb.quantize_model(params)
net = pb.build_network(qm)
rng = np.random.default_rng(1)
for l in (10, 50, 100):
    src = rng.integers(3, 32000, l)
    enc = net.encode(src)
    st = net.initial_state(enc, 1)
    y = np.array([2])
    mx = []
    for step in range(6):
        lp, st2, al = net.decoder_step(y, st, enc)
        sp = st2.s_prime
        u = net.attention.state_proj.apply(sp) if hasattr(net.attention, 'state_proj') else None
        if u is None:
            print([a for a in dir(net.attention) if not a.startswith('_')]); break
        x = enc.att_proj + u
        mx.append(float(np.abs(x).max()))
        y = np.array([int(np.argmax(lp[:, 0]))])
        st = st2
    print(l, 'max|ap+u| per step', [round(v, 3) for v in mx], 'max|ap|', float(np.abs(enc.att_proj).max()))
