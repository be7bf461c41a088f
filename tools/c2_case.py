"""A few c2 chunks (249 x 900 x 70) through StreamingRX, for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.stream import StreamingRX
from paper_2602_13509_b200.synth import Scene
L, S, B = 249, 900, 70
sc = Scene(2, S, B, 5)
tabs = P.CalibrationTables(sc.dark, sc.coeff)
raw = sc.generate(0, L * 6)
srx = StreamingRX(tabs, L, 0.99, use_graph=False)
for i in range(6):
    srx.update(raw[i * L:(i + 1) * L])
torch.cuda.synchronize()
print("ok")
