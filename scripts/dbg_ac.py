import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_0904_0939_b200 import kernels
g = np.load('/root/repo/tests/golden/kernels.npz')
for n in (4, 5, 8, 13):
    psi = g[f"n{n}_psi"]; out = psi.copy()
    kernels.stencil_update(psi, g[f"n{n}_coef_a"], g[f"n{n}_coef_c"], out, 1, n)
    want = g[f"n{n}_update"]
    d = np.argwhere(out != want)
    print(n, len(d), d[:8].tolist())
    if len(d): 
        i,j,k = d[0]; print('  got', out[i,j,k], 'want', want[i,j,k], 'psi', psi[i,j,k])
