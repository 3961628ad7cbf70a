import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
G = torch.from_numpy(np.load("dbg/G_cfg2.npy")).cuda()
d, e, t = fkk.fkk_debug_tridiag(G)
out = {"d": d.cpu().numpy(), "e": e.cpu().numpy(), "tau": t.cpu().numpy()}
os.environ["FKK_EIG_FORCE_L2"] = "1"
d2, e2, t2 = fkk.fkk_debug_tridiag(G)
out.update({"d2": d2.cpu().numpy(), "e2": e2.cpu().numpy(), "tau2": t2.cpu().numpy()})
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/tridiag_dbg.npz", **out)
dd = np.abs(out["d"] - out["d2"]) / np.abs(out["d2"]).max()
print("first d diff >1e-10 at", np.argmax(dd > 1e-10), dd.max())
ee = np.abs(np.abs(out["e"]) - np.abs(out["e2"])) / np.abs(out["e2"]).max()
print("first e diff >1e-10 at", np.argmax(ee > 1e-10), ee.max())
