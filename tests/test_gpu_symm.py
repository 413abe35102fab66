"""Single-process smoke of the NVLink peer-memory wiring (the
symmetric-memory path had never executed): a world-size-1 NCCL process
group, torch symmetric memory for the packed buffers (dist.symmetric_packed_
buffers), the fused encode + all-gather by peer stores (dist.pushed_encode)
and the pull decode (dist.pulled_decode) -- byte-identical to the plain
encode / decode.  With one rank the "peers" are this GPU's own mapping, so
this proves the rendezvous, the pointers and the kernels' use of them, not
NVLink bandwidth.  Runs in a subprocess so the process group and the
symmetric heap never leak into other tests."""
import os
import subprocess
import sys
import textwrap

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r'''
    import os, socket, sys
    sys.path.insert(0, os.environ["EXMY_ROOT"])
    import torch
    import torch.distributed as dist
    import paper_2405_13938_b200 as exmy
    from paper_2405_13938_b200 import dist as xdist
    import workloads as W

    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    R, C, fmt = 1024, 2048, "e3m3"
    t = W.bf16_weights((R, C), seed=21, device="cuda")
    ref = exmy.encode(t, fmt)
    nb = ref.data.numel()
    buf, peers = xdist.symmetric_packed_buffers(nb)
    assert len(peers) == 1
    buf.zero_()
    meta, sp = xdist.pushed_encode(t, fmt, R, 0, peers)
    torch.cuda.synchronize()
    assert int(meta.item()) == int(ref.meta.item())
    assert torch.equal(buf, ref.data), "pushed bytes != encode"
    out = xdist.pulled_decode(buf, R, C, fmt, meta, peers, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), exmy.decode(ref).view(torch.int16)), "pulled decode != decode"
    mc = xdist.multicast_status(buf)
    mp = xdist.multicast_ptr(buf)
    if mp:
        # NVLS multicast push: one multimem.st per store, same bytes
        buf.zero_()
        torch.cuda.synchronize()
        meta2, _ = xdist.pushed_encode(t, fmt, R, 0, peers, meta=meta, multicast=mp)
        torch.cuda.synchronize()
        assert torch.equal(buf, ref.data), "multicast pushed bytes != encode"
        # fp32 input and a k = 9 format through the multicast stores too
        t32 = W.f32_wide((512, 1024), seed=22).cuda()
        ref32 = exmy.encode(t32, "e4m4")
        buf2, peers2 = xdist.symmetric_packed_buffers(ref32.data.numel())
        mp2 = xdist.multicast_ptr(buf2)
        buf2.zero_()
        xdist.pushed_encode(t32, "e4m4", 512, 0, peers2, meta=ref32.meta, multicast=mp2)
        torch.cuda.synchronize()
        assert torch.equal(buf2, ref32.data), "multicast fp32 e4m4 != encode"
        mc["multicast_push_verified"] = True
    print("SYMM_OK", mc)
    dist.destroy_process_group()
''')


def test_symmetric_memory_push_pull_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, EXMY_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and "SYMM_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    print(r.stdout.strip().splitlines()[-1])
