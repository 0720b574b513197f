"""GPU (one device, two processes): the pair exchange mechanics for real.

Each rank exports its receive buffer and flag words by CUDA IPC
(`hp_alloc` + `hp_ipc_get_handle`), opens the partner's (`hp_ipc_open`), and
pushes a known branch output into the partner's buffer with `hp_stage_send`
(vector stores through the mapped pointer + system-scope release of the step
number). After a host barrier each rank checks the payload and the flag, then
runs the fused sampler kernel with the in-kernel flag wait on an ALREADY
released flag (so no kernel ever waits on another process's kernel — the
rule for sharing one GPU) and the partner's data as eps_u, against torch.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, port, q):
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    try:
        from paper_2602_21760_b200 import _kernels as K, _native as N
        from paper_2602_21760_b200.parallel import PeerBuffers, _Raw
        lib = N.load()
        n = 65536 + 40
        buf = PeerBuffers(n, 2, None, 1 - rank)
        gen = torch.Generator(device="cuda").manual_seed(100 + rank)
        mine = torch.randn(n, device="cuda", generator=gen).bfloat16()
        s = 7
        # push my branch output into the partner's slot for step s and release the flag
        rc = lib.hp_stage_send(C.c_void_p(buf.peer_slot(s)), C.c_void_p(mine.data_ptr()), n * 2,
                               C.c_void_p(buf.peer_flags + 4 * rank), s, C.c_void_p(N.stream_ptr()))
        assert rc == 0, rc
        torch.cuda.synchronize()
        dist.barrier()
        # what the partner pushed into MY slot
        other = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(100 + 1 - rank)).bfloat16()
        got = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        cp = torch.cuda.current_stream()
        rc = lib.hp_stage_send(C.c_void_p(got.data_ptr()), C.c_void_p(buf.local_slot(s)), n * 2, None, 0,
                               C.c_void_p(cp.cuda_stream))
        assert rc == 0
        flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        rc = lib.hp_stage_send(C.c_void_p(flags.data_ptr()), C.c_void_p(buf.flags), 16, None, 0,
                               C.c_void_p(cp.cuda_stream))
        assert rc == 0
        ok_payload = bool(torch.equal(got, other))
        ok_flag = int(flags[1 - rank].item()) == s
        # fused sampler with the in-kernel flag acquire (flag already released) and the
        # partner's data read straight from this rank's receive buffer
        x = torch.randn(n, device="cuda")
        out = torch.empty_like(x)
        eps_c, eps_u = (mine, _Raw(buf.local_slot(s), n, torch.bfloat16, x.device)) if rank == 0 else \
            (_Raw(buf.local_slot(s), n, torch.bfloat16, x.device), mine)
        K.sampler_step(x=x, eps_c=eps_c, eps_u=eps_u, x_out=out, update=N.HP_UPDATE_EULER, dt=0.05, w=2.0,
                       wait_flag=buf.flags + 4 * (1 - rank), wait_value=s)
        ec = (mine if rank == 0 else other).float()
        eu = (other if rank == 0 else mine).float()
        ref = x - (ec + 2.0 * (ec - eu)) * 0.05
        ok_step = float((out - ref).abs().max()) < 1e-5
        q.put((rank, ok_payload, ok_flag, ok_step))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ipc_push_flag_and_fused_wait_on_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(_port(), q), nprocs=2, join=True, start_method="spawn")
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, ok_payload, ok_flag, ok_step in res:
        assert ok_payload, f"rank {rank}: payload over IPC differs"
        assert ok_flag, f"rank {rank}: flag not released"
        assert ok_step, f"rank {rank}: fused step with peer operand differs"
