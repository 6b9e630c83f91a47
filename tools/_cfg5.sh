cd $GRAFT_REPO_ROOT
for p in 1 2 3 4 5; do
  timeout 900 python tools/time_setup.py --cells 48 --degree $p --levels 3 --radius 0.5 --solve omg --max-it 3000 2>/dev/null | tail -1
done
