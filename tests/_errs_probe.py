import sys, torch, numpy as np
sys.path.insert(0, '.')
import oracle as O
from tests.test_gpu_parity import _run_layer
from tests._util import normwise, f64, i64
import paper_2601_05296_b200 as M
for (T,d,h,E,k,dt,rn,rt) in [(512,256,384,8,2,"bf16",False,"balanced"),(2048,512,768,8,2,"bf16",False,"skewed"),(3000,256,1408,64,6,"bf16",False,"balanced"),(4096,1024,512,16,2,"bf16",True,"balanced")]:
    inp,out=_run_layer(M,T,d,h,E,k,dt,rn,rt)
    X,WG,W1,W2,W3,DY=(f64(inp[n]) for n in ("x","w_gate","w1","w2","w3","dy"))
    fwd=O.layer_forward(X,WG,W1,W2,W3,k,rn,logits=f64(out["logits"]))
    bwd=O.layer_backward(fwd,DY,X,WG,W1,W2,W3,rn)
    e={n:round(normwise(out[n],fwd[n] if n in ("A","B","y") else bwd[n]),5) for n in ("A","B","y","dA","dB","dg","dx","dw1","dw2","dw3","dw_gate")}
    print((T,d,h,E,k), e, flush=True)
