"""Time one integrate of the DRM19-class flame field (L^3 cells) with the kernel given; prints cells/s.
Library from BDFB_LIB (experiment variants) or the in-tree build."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_01713_b200 as P
from synth import flame_field
L = int(sys.argv[1]) if len(sys.argv) > 1 else 96
kernel = sys.argv[2] if len(sys.argv) > 2 else "thread"
mech = sys.argv[3] if len(sys.argv) > 3 else "drm19"
name, n = {"drm19": ("drm19_class", 22), "h2": ("h2_lidryer", 10)}[mech]
y, rho, F, prog = flame_field(name, L)
dev = torch.device("cuda", 0)
b = P.Batch(y.shape[1], n, 1e-6, 1e-10)
b.set_kernel(kernel)
b.set_model(mech)
Yd, Fd, Rd = torch.tensor(y, device=dev), torch.tensor(F, device=dev), torch.tensor(rho, device=dev)
for r in range(2):
    yy = Yd.clone()
    b.integrate(0.0, 1e-5, yy, f_ext=Fd, aux=Rd)
    st = b.stats()
    ms = b.last_kernel_ms()
print(f"{os.environ.get('BDFB_LIB', 'in-tree').split('/')[-1]} {mech} {kernel} L={L}: {ms:.1f} ms "
      f"{y.shape[1] / ms * 1e3:.4g} cells/s nst={st['nst']} nfe={st['nfe']} failed={st['n_failed']}", flush=True)
