"""Timing of the layer mixer (phalanx_layer_mix*) over group counts and logit flags,
back to back, against the plain mixer: python tools/layer_time.py [B L H D]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import layer_inputs

B, L, H, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 4096, 16, 128)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def b2b(fn, n=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = E(), E()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


g = {k: v.cuda() for k, v in layer_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
print(f"B={B} L={L} H={H} D={D}")
for path in (P.SWR_PATH_AUTO, P.SWR_PATH_FFMA):
    P.set_path(path)
    t = b2b(lambda: P.phalanx_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"]))
    print(f"path {path} phalanx_mix_bwd {t:.1f} us (last path {P.last_path()})", flush=True)
    for G in (H, H // 2, max(H // 8, 1)):
        gg = {k: v.cuda() for k, v in layer_inputs(B, L, H, D, G, G, dtype=torch.bfloat16, seed=1).items()}
        for la, lk in ((False, False), (True, True)):
            try:
                tf = b2b(lambda: P.phalanx_layer_mix(gg["q"], gg["zk"], gg["v"], gg["za"], logit_a=la, logit_k=lk))
                tb = b2b(lambda: P.phalanx_layer_mix_bwd(gg["q"], gg["zk"], gg["v"], gg["za"], gg["dy"], logit_a=la,
                                                         logit_k=lk))
                print(f"path {path} G={G} logits={la},{lk}: fwd {tf:.1f} bwd {tb:.1f} us (last path {P.last_path()})",
                      flush=True)
            except P.SwrError as e:
                print(f"path {path} G={G}: {e}")
