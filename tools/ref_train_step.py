"""CPU timing of the reference's own training step for one view (render_forward +
L1/SSIM loss gradients + render_backward with its compiled kernels), for the
GPU/CPU comparison in profiles/r1_train_step.jsonl.  Needs /root/reference
(this container only) and `make -C oracle ref`.  Usage: python tools/ref_train_step.py C2
"""
import sys, time, numpy as np
ROOT = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + '/tests/golden')
import make_golden as mg
ss = mg.import_reference()
from splatstream import rasterizer as R, metrics as M, model as MD, camera as C
from paper_2512_20943_b200 import synth
cfg = synth.CONFIGS[sys.argv[1]]
c0 = synth.cameras(cfg)[0]
cam = C.Camera(pose=c0.pose, focal=c0.focal, resolution=c0.resolution) if hasattr(C,'Camera') else None
params = synth.Sequence(cfg, seed=0, event_every=0).frame(0)
f = MD.GaussianFrame(params=params)
rng = np.random.default_rng(0)
target = rng.uniform(0,1,(c0.resolution[1], c0.resolution[0], 3))
t0=time.time()
img, st = R.render_forward(f, cam)
t1=time.time()
d = 0.8*M.l1_grad(img, target) - 0.1*M.ssim_grad(img, target)
t2=time.time()
g = R.render_backward(st, d)
t3=time.time()
print(sys.argv[1], 'forward %.2f s, loss grads %.2f s, backward %.2f s, total %.2f s'%(t1-t0,t2-t1,t3-t2,t3-t0))
