import os, sys
sys.path.insert(0, "/root/repo")
import __graft_entry__
__graft_entry__.build()
import torch
from paper_1805_01772_b200 import cf
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device
from synth import rnn_inputs
T,B,I,H,L = 5,2,4,8,1
f = rnn_inputs(T,B,I,H,L, seed=0, len_mode="full")
p = dynamic_rnn_lstm(T,B,I,H,L)
s = cf.Session(p.g, p.fetch_tensors())
print(s.describe())
try:
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    print("ok", tr["pushes"], tr["pops"])
except Exception as e:
    print("ERR", e)
