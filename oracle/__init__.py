"""CPU fp64 oracle for arXiv 1805.01772 ("Dynamic Control Flow in Large-Scale Machine
Learning", Yu et al.).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under ``oracle/``. The
product path (``paper_1805_01772_b200``, ``libcf``) never imports, links or executes it and
shares no code with it; the only shared module is the seeded input generator ``synth``.

What it is: a plain, slow, single-process tagged-token dataflow interpreter in float64
(numpy), written from the paper:

* ``graph``    -- IR + builder: ``cond`` / ``while_loop`` compiled to the five primitives
                  (§4.2), TensorArrays (§2.1), the hidden
                  loop counter (§5.1 feature 1).
* ``kernels``  -- fp64 op kernels (MatMul, elementwise, fused LSTMCell and its gradient).
* ``interp``   -- the local executor (§4.3) implementing the evaluation
                  rules of Fig. "Evaluation rules", dead propagation
                   and the parallel-iterations window.
* ``autodiff`` -- ``gradients`` (§5.1 four-step algorithm) with cond
                  gradients, while-loop gradients,
                  stack-based state saving, predicate stacks for
                  cond-in-while and TensorArray duality
                  (PAPER.md:1110-1131).
* ``models``   -- the dynamic_rnn LSTM workload and the
                  random-projection loss (SURVEY.md §8(c) C-amb 11).

Pins (tests/test_oracle_*.py): closed forms of the paper's loop example, static unrolling,
``torch.nn.LSTM`` (float64, a library routine), central finite differences, brute-force
enumeration of cond branches, and the invariants the paper fixes. No function here is
"parity unpinned".
"""
