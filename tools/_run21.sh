cd $GRAFT_REPO_ROOT
# session 5, call 6: steady-state launch lists of the cfg2 solves with the new defaults (host-decision drivers: same kernels, visible to ncu one by one)
XDG_OMG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2_omg_cfg2_steady.csv python tools/profile_solve.py tests/golden/large/cfg2.npz omg 600 --steady > gpurun_out/ncu_omg.log 2>&1
python tools/launch_summary.py gpurun_out/r2_omg_cfg2_steady.csv | tee gpurun_out/r2_omg_cfg2_steady600_summary.txt | head -n 30
XDG_GMRES_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2_gmres_cfg2_steady.csv python tools/profile_solve.py tests/golden/large/cfg2.npz gmres 60 --steady > gpurun_out/ncu_gmres.log 2>&1
python tools/launch_summary.py gpurun_out/r2_gmres_cfg2_steady.csv | tee gpurun_out/r2_gmres_cfg2_steady60_summary.txt | head -n 20
rm -f gpurun_out/r2_omg_cfg2_steady.csv
