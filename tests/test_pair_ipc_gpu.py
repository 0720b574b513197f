"""GPU (one device, three processes): the group exchange mechanics for real.

Each rank exports its receive slots and flag words by CUDA IPC
(`hp_alloc` + `hp_ipc_get_handle`, ``parallel.LinkBuffers``), opens the
others' (`hp_ipc_open`), and pushes a known branch output as message 1 of its
link to every other rank (`hp_stage_broadcast`: vector stores through the
mapped pointer + system-scope release of the link's message count into the
destination's flag). Rank 2 also acknowledges message 1 to ranks 0 and 1.
After a host barrier each rank checks payloads, flags (read from the host with
`hp_flag_poll`) and acks, then runs the fused sampler kernel with the
in-kernel flag wait on ALREADY released flags (so no kernel ever waits on
another process's kernel — the rule for sharing one GPU) and remote operands
read from its receive slots, against torch.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 3


def _payload(src, n):
    g = torch.Generator(device="cuda").manual_seed(100 + src)
    return torch.randn(n, device="cuda", generator=g).bfloat16()


def _worker(rank, port, q):
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    try:
        from paper_2602_21760_b200 import _kernels as K, _native as N
        from paper_2602_21760_b200.parallel import LinkBuffers, _Raw
        lib = N.load()
        n = 65536 + 40
        buf = LinkBuffers(n * 2, None, rank, WORLD)
        mine = _payload(rank, n)
        s = 1                                   # message 1 on every link
        others = [r for r in range(WORLD) if r != rank]
        dsts = (C.c_void_p * len(others))(*[buf.peer_slot(r, s) for r in others])
        flags = (C.c_void_p * len(others))(*[buf.peer_data_flag(r) for r in others])
        rc = lib.hp_stage_broadcast(dsts, flags, len(others), C.c_void_p(mine.data_ptr()), n * 2, s,
                                    C.c_void_p(N.stream_ptr()))
        assert rc == 0, rc
        if rank == 2:       # rank 2 consumed message 1 of ranks 0 and 1: acknowledge
            acks = (C.c_void_p * 2)(buf.peer_ack_flag(0), buf.peer_ack_flag(1))
            rc = lib.hp_stage_broadcast((C.c_void_p * 2)(0, 0), acks, 2, None, 0, s, C.c_void_p(N.stream_ptr()))
            assert rc == 0, rc
        torch.cuda.synchronize()
        dist.barrier()
        st = C.c_void_p(N.stream_ptr())
        ok_payload = True
        for src in others:
            got = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            assert lib.hp_stage_send(C.c_void_p(got.data_ptr()), C.c_void_p(buf.local_slot(src, s)), n * 2,
                                     None, 0, st) == 0
            ok_payload &= bool(torch.equal(got, _payload(src, n)))
        fl = torch.zeros(16, dtype=torch.int32, device="cuda")
        assert lib.hp_stage_send(C.c_void_p(fl.data_ptr()), C.c_void_p(buf.flags), 64, None, 0, st) == 0
        fl = fl.tolist()
        got = C.c_uint32()
        ok_flag = all(fl[src] == s for src in others) and fl[rank] == 0
        ok_flag &= all(lib.hp_flag_poll(C.c_void_p(buf.data_flag(src)), s, 1_000_000_000, C.byref(got)) == 0
                       and got.value == s for src in others)
        ok_ack = buf.ack_flag(2) and fl[WORLD + 2] == s if rank < 2 else True
        # fused sampler: remote operands straight from this rank's receive buffer
        x = torch.randn(n, device="cuda")
        out = torch.empty_like(x)
        remote = {src: _Raw(buf.local_slot(src, s), n, torch.bfloat16, x.device) for src in others}
        ops = {rank: mine, **remote}
        if rank == 2:
            assert lib.hp_flag_wait(C.c_void_p(buf.data_flag(0)), s, None, 1_000_000_000, st) == 0
        K.sampler_step(x=x, eps_c=ops[0], eps_u=ops[1], x_out=out, update=N.HP_UPDATE_EULER, dt=0.05, w=2.0,
                       wait_flag=buf.data_flag(1 if rank != 1 else 0), wait_value=s)
        ec, eu = _payload(0, n).float(), _payload(1, n).float()
        ref = x - (ec + 2.0 * (ec - eu)) * 0.05
        ok_step = float((out - ref).abs().max()) < 1e-5
        q.put((rank, ok_payload, ok_flag, ok_ack, ok_step))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ipc_broadcast_flags_acks_and_fused_wait_on_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(_port(), q), nprocs=WORLD, join=True, start_method="spawn")
    res = sorted(q.get(timeout=10) for _ in range(WORLD))
    for rank, ok_payload, ok_flag, ok_ack, ok_step in res:
        assert ok_payload, f"rank {rank}: payload over IPC differs"
        assert ok_flag, f"rank {rank}: flag not released"
        assert ok_ack, f"rank {rank}: passive rank's acknowledgement missing"
        assert ok_step, f"rank {rank}: fused step with peer operand differs"
