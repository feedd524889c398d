python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'P'
import json; d=json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("factor", round(d["factor_ms"],2), "solve", round(d["solve_ms"],3), "q32", round(d["solve_ms_q32"],2), "resid", d["residual"], "e2e", round(d["e2e"]["factor_ms"],1), round(d["e2e"]["solve_ms"],1))
print("levels", [round(x,2) for x in d["level_ms"]]); print(d["factor_phase_ms_eager"])
P
