"""CPU cost of one graph-replayed decode step (hx_decode_step_device) vs its GPU
time, and the synchronous host-token call (hx_decode_step): where the e2e gap
comes from. python tools/launch_cost.py [layers] [context]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    import torch
    import paper_2507_07120_b200 as P
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    spec = P.model.PRESETS["llama3-8b-like"]
    B = 8
    eng = P.HelixDecoder(spec, tpa=1, kvp=1, batch=B, capacity=S + 4096, layers=L)
    eng.init_weights(2507, qkv="hash")
    eng.fill_kv_hash(S, 2507)
    tok = [torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda"),
           torch.zeros(B, dtype=torch.int32, device="cuda")]
    for i in range(5):
        eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
    eng.synchronize()
    n = 50
    t0 = time.perf_counter()
    for i in range(n):
        eng.step_device(tok[i % 2].data_ptr(), tok[(i + 1) % 2].data_ptr())
    t1 = time.perf_counter()
    eng.synchronize()
    t2 = time.perf_counter()
    cpu_launch = (t1 - t0) / n * 1e3
    gpu = (t2 - t0) / n * 1e3
    h_tok = torch.zeros(B, dtype=torch.int32).pin_memory()
    h_next = torch.zeros(B, dtype=torch.int32).pin_memory()
    ip = ctypes.POINTER(ctypes.c_int32)
    for i in range(3):
        P._lib.check(P.lib().hx_decode_step(eng._h, ctypes.cast(h_tok.data_ptr(), ip), ctypes.cast(h_next.data_ptr(), ip),
                                            None, None), eng._h)
    t3 = time.perf_counter()
    for i in range(n):
        P._lib.check(P.lib().hx_decode_step(eng._h, ctypes.cast(h_tok.data_ptr(), ip), ctypes.cast(h_next.data_ptr(), ip),
                                            None, None), eng._h)
        h_tok.copy_(h_next)
    t4 = time.perf_counter()
    print(f"layers {L} ctx {S}: graph launch CPU {cpu_launch:.3f} ms/step, pipelined {gpu:.3f} ms/step, "
          f"synchronous host-token step {(t4 - t3) / n * 1e3:.3f} ms/step, kernels/step {eng.info()['kernels_per_step']}")
    eng.close()


if __name__ == "__main__":
    main()
