import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import chase_inputs as ci, oracle
import paper_2309_15595_b200 as cb
from gpu_util import dev, host
N, n, complex_ = 300, 64, False
lam = ci.uniform_spectrum(N, -2.0, 3.0)
A = ci.dense_from_spectrum(lam, N + n, complex_)
C, _ = np.linalg.qr(ci.gaussian_block(N, n, N + 1, complex_))
Q = C.conj().T @ A @ C
os.environ["CHASE_HEEVD_DUMP"] = "gpurun_out/dump.txt"
h = cb.Chase(cb.CHASE_R64, N, n)
Ad, Cd = dev(A), dev(np.asfortranarray(C))
theta, sw = h.rayleigh_ritz(Ad, Cd)
torch.cuda.synchronize()
np.save("gpurun_out/Q.npy", Q)
print("theta err", np.max(np.abs(theta - np.linalg.eigvalsh(Q))))
