"""Host-side overhead of one pipeline step (perf_counter around each call, no syncs)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2506_19656_b200 import pipeline, synth, _lib
from paper_2506_19656_b200 import _device as dev

d = torch.device('cuda', 0)
x = synth.minicube(19656, (495, 128, 128, 7), device=d)
spec = pipeline.StreamSpec(8)
recon = torch.empty(x.shape, dtype=torch.float32, device=d)
for _ in range(3):
    enc = pipeline.encode_prep(x, spec); pipeline.decode_eval(enc, x, recon_out=recon, want_ssim=False)
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(10):
    enc = pipeline.encode_prep(x, spec); pipeline.decode_eval(enc, x, recon_out=recon, want_ssim=False)
pr.disable()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3*(t1-t0)/10:.3f} ms/step, total {1e3*(t2-t0)/10:.3f} ms/step")
pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
