"""Factorization time (graph replay, device-resident) under several settings of
the tuning switches, each in its own process (process-wide switches such as
KS_PDL are read once). The config's operator is produced once and cached in
the library's operator file format under /tmp.

    python tools/sweep_factor.py "" "KS_GROUPS=4" "KS_PDL=0 KS_GROUPS=16" ...
    CFG=cfg4 python tools/sweep_factor.py ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(path: str, lam: float, reps: int) -> None:
    import numpy as np
    import torch

    import paper_1602_01376_b200 as ks

    prob = ks.load_operator(path)
    st = torch.cuda.current_stream()
    hf = ks.factorize(prob, lam)
    for _ in range(3):
        hf.refactorize(lam, st.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hf.refactorize(lam, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    b = torch.ones(hf.n, 1, dtype=torch.float64, device="cuda")
    x = ks.solve_many(hf, b)
    r = ks.hss_matvec(hf, x) + lam * x - b
    print(json.dumps({"mean": float(np.mean(ts)), "min": float(np.min(ts)),
                      "resid": float(torch.linalg.norm(r) / torch.linalg.norm(b))}), flush=True)


def main():
    from paper_1602_01376_b200.configs import CONFIGS

    cfg = CONFIGS[os.environ.get("CFG", "cfg3")]
    path = f"/tmp/ks_op_{cfg.name}.ksop"
    if not os.path.exists(path):  # in a child process: its GPU memory is gone before the workers run
        subprocess.run([sys.executable, __file__, "--produce", cfg.name, path], check=True, timeout=1800)
    for setting in sys.argv[1:] or [""]:
        env = dict(os.environ)
        for kv in setting.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--worker", path, str(cfg.lam)], env=env, capture_output=True,
                             text=True, timeout=600)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(f"[{setting or 'default'}] {line}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--worker":
        worker(sys.argv[2], float(sys.argv[3]), 7)
    elif len(sys.argv) > 1 and sys.argv[1] == "--produce":
        import paper_1602_01376_b200 as ks
        from paper_1602_01376_b200.configs import CONFIGS
        from producer import make_operator

        ks.save_operator(make_operator(CONFIGS[sys.argv[2]], device="cuda"), sys.argv[3])
    else:
        main()
