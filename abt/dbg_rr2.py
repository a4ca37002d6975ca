import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import chase_inputs as ci
import paper_2309_15595_b200 as cb
from gpu_util import dev, host
def run(N, n, complex_, tag):
    lam = ci.uniform_spectrum(N, -2.0, 3.0)
    A = ci.dense_from_spectrum(lam, N + n, complex_)
    C, _ = np.linalg.qr(ci.gaussian_block(N, n, N + 1, complex_))
    Q = C.conj().T @ A @ C
    os.environ["CHASE_HEEVD_DUMP"] = f"gpurun_out/dump_{tag}.txt"
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n)
    Ad, Cd = dev(A), dev(np.asfortranarray(C))
    theta, sw = h.rayleigh_ritz(Ad, Cd)
    torch.cuda.synchronize()
    h.close()
    print(tag, N, n, complex_, "theta err", np.max(np.abs(theta - np.linalg.eigvalsh(Q))), flush=True)
for tag, (N, n, c) in enumerate([(64,1,True),(64,1,False),(64,7,True),(64,7,False),(200,60,True),(200,60,False),(300,64,True),(300,64,False),(300,64,False),(301,65,True),(301,65,False)]):
    run(N, n, c, tag)
