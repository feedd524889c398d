"""Times one LU panel launch (k_lu_panel2) on
random nodes and prints CTA 0's phase clocks (ks_probe_panel)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1602_01376_b200", "libinvaskit.so"))
for T, tp, w, cnt in [(768, 512, 16, 1), (768, 512, 16, 16), (768, 512, 16, 256), (768, 512, 32, 1), (1536, 1024, 8, 1)]:
    ms = (C.c_double * 2)()
    clk = (C.c_longlong * 64)()
    rc = lib.ks_probe_panel(T, tp, w, cnt, 20, ms, clk)
    c = list(clk)
    base = c[0]
    st = {i: c[i] - base for i in list(range(24)) + list(range(26, 46)) if c[i]}
    print(f"T={T} tp={tp} w={w} count={cnt} rc={rc} min {ms[0]*1e3:.1f} us med {ms[1]*1e3:.1f} us moves={c[24]}")
    print("   stamps (cycles from start):", st)
