"""Independent pin for the oracle's LSTM: torch.nn.LSTM (float64, a library routine) run
one sequence at a time on its unpadded length, differentiated by torch.autograd.

Reading R9 (gate order i,f,g,o; W = [W_ih | W_hh]; b_ih = b, b_hh = 0) and R10 (a finished
row keeps its state and emits zeros) make this an independent computation of exactly what
the oracle's dynamic_rnn program computes. Not used by the product path.
"""
import numpy as np
import torch


def torch_dynamic_rnn(f, T, B, I, H, L):
    torch.manual_seed(0)
    x = torch.tensor(f["x"], requires_grad=True)
    lens = [int(v) for v in f["len"]]
    inp = x
    y = torch.zeros((), dtype=torch.float64)
    mods, h0s, c0s, hTs, cTs = [], [], [], [], []
    for l in range(L):
        il = I if l == 0 else H
        m = torch.nn.LSTM(il, H, dtype=torch.float64)
        W = f[f"W{l}"]
        with torch.no_grad():
            m.weight_ih_l0.copy_(torch.tensor(W[:, :il]))
            m.weight_hh_l0.copy_(torch.tensor(W[:, il:]))
            m.bias_ih_l0.copy_(torch.tensor(f[f"b{l}"]))
            m.bias_hh_l0.zero_()
        h0 = torch.tensor(f[f"h0_{l}"], requires_grad=True)
        c0 = torch.tensor(f[f"c0_{l}"], requires_grad=True)
        outs, hs, cs = [], [], []
        for bi in range(B):
            n = lens[bi]
            if n == 0:
                outs.append(torch.zeros(T, H, dtype=torch.float64))
                hs.append(h0[bi])
                cs.append(c0[bi])
                continue
            o, (hn, cn) = m(inp[:n, bi:bi + 1], (h0[bi:bi + 1][None], c0[bi:bi + 1][None]))
            outs.append(torch.cat([o[:, 0], torch.zeros(T - n, H, dtype=torch.float64)]))
            hs.append(hn[0, 0])
            cs.append(cn[0, 0])
        out = torch.stack(outs, 1)
        hT, cT = torch.stack(hs), torch.stack(cs)
        y = y + (torch.tensor(f[f"R_h{l}"]) * hT).sum() + (torch.tensor(f[f"R_c{l}"]) * cT).sum()
        mods.append(m)
        h0s.append(h0)
        c0s.append(c0)
        hTs.append(hT)
        cTs.append(cT)
        inp = out
    y = y + (torch.tensor(f["R_out"]) * out).sum()
    y.backward()
    res = {"y": y.item(), "out": out.detach().numpy(), "dx": x.grad.numpy()}
    for l, m in enumerate(mods):
        res[f"hT{l}"] = hTs[l].detach().numpy()
        res[f"cT{l}"] = cTs[l].detach().numpy()
        res[f"dW{l}"] = np.concatenate([m.weight_ih_l0.grad.numpy(), m.weight_hh_l0.grad.numpy()], 1)
        res[f"db{l}"] = m.bias_ih_l0.grad.numpy()
        res[f"dh0_{l}"] = h0s[l].grad.numpy()
        res[f"dc0_{l}"] = c0s[l].grad.numpy()
    return res
