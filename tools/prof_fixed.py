import os, sys
sys.path.insert(0, os.getcwd())
import torch, bgk_inputs as bi
from paper_2408_02350_b200 import Bgk
cfg = bi.C5.replace(ale=0, manage=0)
g = Bgk(cfg, bi.make_cloud(cfg), device="cuda:0")
g.step(3); g.sync(); torch.cuda.synchronize(); print("done")
