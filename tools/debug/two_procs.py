"""Two processes sharing one GPU, each running dc_correct on its own 512-pulse C4 shard (diagnostics for
the two-ranks-on-one-GPU failure).  python tools/debug/two_procs.py [gloo|none] [lib.so|-] [correct20|iono20|iono16|doppler20|...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def work(rank, mode, lib, port, q, what):
    import numpy as np
    import torch
    import paper_2508_04951_b200 as dc
    import synth
    if lib:
        dc.use_library(lib)
    if mode == "gloo":
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    npul = 512
    if "x" in what:  # e.g. correct20x256: 256 pulses per process
        what, npul = what.split("x")[0], int(what.split("x")[1])
    log2n = int(what[-2:])
    n, pulses = 1 << log2n, npul * (1 << 20) // (1 << log2n)
    bank = synth.waveform_bank(n, count=16)
    idx = (np.arange(pulses) + pulses * rank) % 16
    x = torch.from_numpy(bank[idx]).cuda()
    y = torch.empty_like(x)
    tec, alpha = synth.pulse_params(2 * pulses)
    tec, alpha = tec[pulses * rank:pulses * (rank + 1)].copy(), alpha[pulses * rank:pulses * (rank + 1)].copy()
    p = dc.Plan(n, 2.048e9, 0.0, taps=32, stream=torch.cuda.current_stream())
    try:
        for _ in range(6):
            if what.startswith("correct"):
                p.correct(x, y, tec, alpha)
            elif what.startswith("seq"):  # the two stages as separate calls on the user's buffers
                p.iono(x, tec)
                p.doppler(x, y, alpha)
            elif what.startswith("iono"):
                p.iono(x, tec)
            elif what.startswith("pq"):
                p.doppler_pq(x, y, alpha)
            else:
                p.doppler(x, y, alpha)
        torch.cuda.synchronize()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"FAIL {e}"))


if __name__ == "__main__":
    import multiprocessing as mp
    import socket
    mode = sys.argv[1] if len(sys.argv) > 1 else "none"
    lib = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else ""
    what = sys.argv[3] if len(sys.argv) > 3 else "correct20"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=work, args=(r, mode, lib, port, q, what)) for r in range(2)]
    for pr in ps:
        pr.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for pr in ps:
        pr.join()
    print(mode, os.path.basename(lib) or "default", what, res)
