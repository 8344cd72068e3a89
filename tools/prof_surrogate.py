import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2109_05948_b200.rng import TAG_TRAIN, Stream
from paper_2109_05948_b200.surrogate import SurrogateNet
n, k, p, K = 1000, 83, 4096, 16
net = SurrogateNet(n, problem="col", arch="small", seed=1)
cands = torch.randint(0, k, (p * K, n), dtype=torch.int32, device="cuda")
y = np.random.default_rng(1).random(p) * 100
net.train_generation(cands[:p], y, k, 1, 64, Stream.derive(1, TAG_TRAIN, 0)); net.predict_assigns_device(cands[:2048], k)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
for what in ("train", "predict"):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        if what == "train":
            net.train_generation(cands[:p], y, k, 1, 64, Stream.derive(1, TAG_TRAIN, 0))
        else:
            net.predict_assigns_device(cands, k)
        torch.cuda.synchronize()
    print(what)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
