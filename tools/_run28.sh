cd $GRAFT_REPO_ROOT
# session 5, call 13: cfg5 p=3 at 48^3 -- OMG iteration count with dense vs multifrontal Schwarz factors (roundoff sensitivity)
for mode in dense sparse; do
echo "== XDG_LOW_ORDER=$mode"
XDG_LOW_ORDER=$mode timeout 900 python tools/time_setup.py --cells 48 --degree 3 --radius 0.5 --solve omg 2>&1 | grep "^{" | tail -n 1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); o = d['omg']
print(d['degree'], d['raw_dofs'], o['iterations'], o['solve_s'], round(o['dof_per_s']), o['converged'], o['final_residual'])"
done | tee gpurun_out/r2_cfg5_p3_48_modes.txt
CELLS=96 PROFILE_SORT=tottime PROFILE_LINES=24 timeout 1500 python tools/profile_setup_solve.py cfg4-native omg 2>&1 | grep -v Warning > gpurun_out/r2_cfg4_sparse_setup_prof_v3.txt
head -n 34 gpurun_out/r2_cfg4_sparse_setup_prof_v3.txt | cut -c1-170
