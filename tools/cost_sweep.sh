# per-side cost-weight sweep of the window partition (WBX_WIN_COST_A / _T = "segment,nonzero")
for ca in 4,1 8,1 12,1; do for ct in 4,1 8,1 12,1; do
  echo "A=$ca T=$ct $(WBX_WIN_COST_A=$ca WBX_WIN_COST_T=$ct python tools/probe_solver.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["tau only (200 power iters)"], d["fista 100 (tau given)"])')"
done; done
