cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== default"; python tools/probe_ns.py --config ns2000 2>&1 | tail -1
echo "== no PDL"; TGA_NS_NO_PDL=1 python tools/probe_ns.py --config ns2000 2>&1 | tail -1
echo "== RW=8"; TGA_NS_RW=8 python tools/probe_ns.py --config ns2000 2>&1 | tail -1
for env in "" "TGA_NS_NO_PDL=1" "TGA_NS_RW=8" "TGA_NS_RW=4"; do
  echo "== sweep $env"; env $env python tools/sweep_time.py --config ns2000 2>&1 | tail -2
done
echo "== sweep cfg2"; python tools/sweep_time.py --config cfg2 2>&1 | tail -2
