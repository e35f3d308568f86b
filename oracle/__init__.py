"""ORACLE — test infrastructure only.

CPU restatements used as the checker by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.  The product
package ``paper_2505_10259_b200`` never imports anything from here.

  accept_ref   C restatement (csrc/accept_oracle.c) of the K7 accept/reject
               step + the acceptance statistics of specpipe/acceptance.py
  model_ref    NumPy target/draft forward (HF-pinned, tests/golden/hf_tiny.npz)
  decode_ref   the dual-batch speculative decoding loop, token for token

Parity status: the accept/reject step and the acceptance statistics are
pinned (reference golden vectors in tests/golden/ref_specpipe.json); model
arithmetic is pinned to transformers (third-party, not in /root/reference);
full-decode token streams are unpinned by the reference itself, which has no
model.
"""
