"""C5 real-time mode, both frame variants back to back (bench.realtime):
zero-copy (kernels on pinned, device-mapped host memory) and explicit copies.

    python tools/rt_bench.py [spots_per_frame] [frames]"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    args = types.SimpleNamespace(rt_spots=int(sys.argv[1]) if len(sys.argv) > 1 else 50,
                                 rt_frames=int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
    for zc in (True, False, True, False):
        r = bench.realtime(args, "cuda:0", zero_copy=zc)
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items() if k != "span"}),
              flush=True)
