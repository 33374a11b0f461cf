"""Per-iteration kernel durations from an ncu launch list (gpu__time_duration.sum, csv)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
for hi, r in enumerate(rows):
    if 'Kernel Name' in r: break
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki].split('(')[0].split('::')[-1].split('<')[0], float(r[vi]) / 1e3) for r in rows[hi + 1:]]
# last cil_icp_run: the last run_init_kernel onwards
last = max(i for i, (k, _) in enumerate(seq) if k == 'run_init_kernel')
it, cur = [], {}
for k, us in seq[last + 1:]:
    if k in ('icp_select_kernel', 'icp_nn_kernel', 'icp_acc_kernel', 'icp_reduce_kernel'):
        cur[k] = us
        if k in ('icp_acc_kernel', 'icp_reduce_kernel'):
            it.append(cur); cur = {}
for n, c in enumerate(it):
    print(f"{n:3d} sel {c.get('icp_select_kernel', 0):8.1f} nn {c.get('icp_nn_kernel', 0):8.1f} "
          f"acc/reduce {c.get('icp_acc_kernel', c.get('icp_reduce_kernel', 0)):7.1f}")
