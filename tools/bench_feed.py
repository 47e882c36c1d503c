"""Throughput of the rows either side of the step on AlexNet-227
b256 bf16, one GPU: the trainer loop `train()` (`pkg/src/parconv/trainer.py:99-154`)
with the HBM-resident split and the on-device batch gather, against the same loop
feeding host batches; `evaluation_errors` (`schemes.py:600-645`) on 256-image test
shards; and the on-device synthetic data generator vs the host one. Prints one JSON
line. python tools/bench_feed.py [epochs]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1312_5853_b200 as P  # noqa: E402
from paper_1312_5853_b200.data import Dataset, synthetic_rows, synthetic_rows_device  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 4
net = P.load_network(ROOT / "configs" / "alexnet.net")
n = 1024          # 4 batches of 256 per epoch
out = {"workload": "AlexNet-227 d1m1 b256 bf16", "images": n, "epochs": epochs}

# synthetic data: device generator vs the host restatement (same values, data.py:52-96)
idx = np.arange(n) % 1000
torch.cuda.synchronize()
t0 = time.perf_counter()
dev = synthetic_rows_device(1000, 2, net.input_shape, 0, np.arange(n))
torch.cuda.synchronize()
out["synthetic_device_images_per_s"] = n / (time.perf_counter() - t0)
t0 = time.perf_counter()
host, labels = synthetic_rows(1000, 2, net.input_shape, 0, np.arange(64))
out["synthetic_host_images_per_s"] = 64 / (time.perf_counter() - t0)
train_set = Dataset(dev.cpu().numpy().astype(np.float64), np.arange(n) // 2, 1000)


def run(device_data: bool):
    cfg = P.TrainConfig(net=net, plan=P.ParallelPlan(1, 1), epochs=epochs, batch=256, seed=0, train_data=train_set,
                        precision="bf16", device_data=device_data, record_wall_time=True,
                        sgd=P.SgdState(learning_rate=0.001))   # He init at lr 0.01 diverges (as in the reference)
    res = P.train(cfg)
    torch.cuda.synchronize()
    w = [r.wall_seconds for r in res.records]
    steps = len(w) - 4          # skip the first 4 steps (engine build, graph capture)
    return 256 * steps / (w[-1] - w[3]), res.records[-1].train_loss


out["train_device_feed_images_per_s"], out["train_loss_last"] = run(True)
out["train_host_feed_images_per_s"], _ = run(False)

# evaluation_errors on 256-image shards of a test split (cached engines after the first call)
fab = P.spawn(1, precision="bf16")
cs = P.columnize(net, 1)
P.setup_workers(fab, P.ParallelPlan(1, 1), cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
tx = train_set.images[:256]
ty = train_set.labels[:256]
P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, tx, ty)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, tx, ty)
out["evaluation_images_per_s"] = 2560 / (time.perf_counter() - t0)
P.hybrid_step(fab, P.ParallelPlan(1, 1), cs, tx, ty)     # after a step: parameters come from the engine
P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, tx, ty)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, tx, ty)
out["evaluation_after_step_images_per_s"] = 2560 / (time.perf_counter() - t0)
txd = torch.as_tensor(np.ascontiguousarray(tx, dtype=np.float32)).cuda()   # device-resident test split
P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, txd, ty)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    P.evaluation_errors(fab, P.ParallelPlan(1, 1), cs, txd, ty)
out["evaluation_device_split_images_per_s"] = 2560 / (time.perf_counter() - t0)
print(json.dumps(out), flush=True)
