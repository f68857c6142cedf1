"""One run of bench.run_server_sample on cuda:0 (quick check of the batcher bench line)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402

p = TfheParams(128)
keys = ClientKeys(p, bench.KEY_SEED)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(p, 0, stream=s.cuda_stream)
ctx.upload_keys(keys.bk, keys.ksk)
print(json.dumps(bench.run_server_sample(ctx, keys, 1, lambda x: x)))
