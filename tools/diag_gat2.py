"""Layer-by-layer GAT backward diagnostic against float64 autograd."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from conftest import rel_l2
from oracle import sage_gat
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200 import ops
from paper_2605_11517_b200.training import TrainSession

F, H, C, L, heads = (int(x) for x in (sys.argv[1:] or [12, 8, 5, 2, 2]))
g = g2.generate_kronecker(9, 8, seed=9)
ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=10)
plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, 4, 1), 4)
model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=12, aggregation_mode="gat", heads=heads)
n = g.num_vertices
graph = sage_gat._graph(g.src_ptr, g.dst_idx)
_, src, dst, _ = graph
loops = torch.arange(n)
s_all, d_all = torch.cat([src, loops]), torch.cat([dst, loops])
x = torch.from_numpy(np.asarray(ds.features, dtype=np.float64))
ws = [torch.tensor(np.asarray(w, dtype=np.float64), requires_grad=True) for w in model.weights]
keep = {}
h = x
for l, wp in enumerate(ws):
    d_in = wp.shape[0] - 2; hd = wp.shape[1]; dh = hd // heads
    W, a_s, a_d = wp[:d_in], wp[d_in].reshape(heads, dh), wp[d_in + 1].reshape(heads, dh)
    P = (h @ W).reshape(n, heads, dh); P.retain_grad()
    s = (P * a_s).sum(-1); t = (P * a_d).sum(-1)
    s.retain_grad(); t.retain_grad()
    z = torch.nn.functional.leaky_relu(s[s_all] + t[d_all], 0.2)
    zmax = torch.full((n, heads), -torch.inf, dtype=z.dtype).scatter_reduce(0, d_all[:, None].expand(-1, heads), z, reduce="amax", include_self=True)
    e = torch.exp(z - zmax[d_all])
    den = torch.zeros((n, heads), dtype=z.dtype).index_add(0, d_all, e)
    al = e / den[d_all]
    O = torch.zeros((n, heads, dh), dtype=z.dtype).index_add(0, d_all, al[..., None] * P[s_all]); O.retain_grad()
    keep[l] = dict(P=P, s=s, t=t, O=O, h=h)
    last = l == L - 1
    h = O.mean(dim=1) if last else torch.relu(O.reshape(n, hd))
loss, acc = sage_gat.masked_xent(h, ds.labels, ds.train_mask)
loss.backward()

sess = TrainSession(ds, plan, model)
eng = sess.engine
eng.g, eng.h = eng._gh
eng.forward(); eng.loss()
print("loss", float(eng.stats[0]), float(loss))
def host(t, cols):
    return t[:, :cols].double().cpu().numpy()
for l in reversed(range(L)):
    c = eng.cfg[l]
    dh, dhp = c.dh, c.dhp
    xin = eng.layer_input(l)
    # emulate _backward_gat up to the gradients
    if c.last:
        go = eng.t2[:, :c.hdp]
        ops.head_mean(eng.g, eng.V, c.heads, c.dh, c.dhp, go, backward=True)
    else:
        go = eng.g[:, :c.hdp]
    gov = host(go, c.hdp).reshape(n, heads, dhp)[:, :, :dh]
    print(f"layer {l} gO", [f"{rel_l2(gov[:, k], keep[l]['O'].grad[:, k].numpy()):.1e}" for k in range(heads)])
    eng._backward_gat(l, xin, 0.0)
    ge = host(eng.h, c.n_ext) if True else None
    gP = ge[:, :c.hdp].reshape(n, heads, dhp)[:, :, :dh]
    print(f"  dP", [f"{rel_l2(gP[:, k], keep[l]['P'].grad[:, k].numpy()):.1e}" for k in range(heads)])
    print(f"  ds", [f"{rel_l2(ge[:, c.hdp + k], keep[l]['s'].grad[:, k].numpy()):.1e}" for k in range(heads)])
    print(f"  dt", [f"{rel_l2(ge[:, c.hdp + heads + k], keep[l]['t'].grad[:, k].numpy()):.1e}" for k in range(heads)])
    if l > 0:
        # dgrad into g (masked by relu of layer l-1 output)
        gp = host(eng.g, c.d_in)
        ref = keep[l - 1]['O'].grad.reshape(n, -1).numpy()
        print(f"  g->layer{l-1}", f"{rel_l2(gp, ref):.1e}")

print("--- weight grads, layer by layer (rerun)")
eng.g, eng.h = eng._gh
eng.forward(); eng.loss()
for l in reversed(range(L)):
    c = eng.cfg[l]
    xin = eng.layer_input(l)
    eng._backward_gat(l, xin, 0.0)
    wt = eng.wts
    d_in, dh, dhp = wt.shape[l]
    X = host(xin, d_in)
    GE = host(eng.h, c.n_ext)
    ref = X.T @ GE
    got = wt.dwext[l][:d_in, :c.n_ext].double().cpu().numpy()
    print(f"layer {l} dwext", f"{rel_l2(got, ref):.1e}", "cols:",
          [f"{rel_l2(got[:, j], ref[:, j]):.0e}" for j in range(c.n_ext)])
    gw = ws[l].grad.numpy()
    dw = wt.dw[l][:d_in].double().cpu().numpy().reshape(d_in, heads, dhp)[:, :, :dh].reshape(d_in, -1)
    print("   dW", f"{rel_l2(dw, gw[:d_in]):.1e}", " datt", f"{rel_l2(wt.datt[l].double().cpu().numpy()[:, :, :dh].reshape(2, -1), gw[d_in:]):.1e}")
