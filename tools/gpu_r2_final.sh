#!/bin/bash
# round-2 final evidence: smoke, full GPU suite, every bench line, launch list + full ncu pages of the
# dominant kernels, reference arm -> gpurun_out/final_*
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final_pytest_gpu.log 2>&1; tail -1 gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err
for spec in "cfg3" "cfg3r2" "cfg4 --no-per-op --steps 20 --warmup 3" "ns2000" "jd" "cfg3f" "cfg5 --no-per-op" \
            "cfg2 --score penalised" "cfg4 --score penalised --no-per-op --steps 20 --warmup 3" "cfg3 --granular 100" "cfg2 --granular 20"; do
  tag=$(echo $spec | awk '{t=$1; for(i=2;i<=NF;i++){ if($i=="--score") t=t"_"$(i+1); if($i=="--granular") t=t"_etga"$(i+1)}; print t}')
  timeout 900 python bench.py --config $spec --no-cpu-baseline > gpurun_out/final_bench_$tag.json 2> gpurun_out/final_bench_$tag.err
  python -c "import json; d=json.loads(open('gpurun_out/final_bench_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$tag us/step %.2f value %.3g kernel %.2f frac %.3f clk %s' % (1e3*d['ms_per_step'], d['value'], 1e3*r['kernel_ms'], r['frac'], (d.get('clocks') or {}).get('sm_mhz')))" || tail -3 gpurun_out/final_bench_$tag.err
done
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inter|k_pick" -c 240 --csv \
  --log-file gpurun_out/final_launches_bench_cfg2.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/final_inter_cfg2 -f python tools/prof_dev.py --config cfg2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pick_update1 -s 4 -c 1 -o gpurun_out/final_pick_cfg2 -f python tools/prof_dev.py --config cfg2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter -s 2 -c 1 -o gpurun_out/final_inter_jd -f python tools/prof_dev.py --config jd --steps 3 > /dev/null 2>&1
for r in final_inter_cfg2 final_pick_cfg2 final_inter_jd; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep gpurun_out/$r.csv; done
ls gpurun_out | grep final | head -50
