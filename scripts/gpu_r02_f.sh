#!/bin/bash
# resident mid-grid solve (sor_tb.cu) + parity + optional bench
TAG=${1:-r02f}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
grep -E "^(FAILED|E )" gpurun_out/pytest_${TAG}.log | head -20
timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}.json > gpurun_out/mid_tb_${TAG}.log 2>&1
python -c "
import json, sys
for r in json.load(open(sys.argv[1])):
    print(r['case'], {k: (round(v['us_per_it'], 2), v['tb_m_used'], v.get('phi_bitwise_equal')) for k, v in r.items() if k.startswith('tb')})
" gpurun_out/mid_tb_${TAG}.json
IBM_SOR_TB=3 ncu --set full --clock-control none --import-source on -k regex:k_sor_tb -c 1 \
    -o gpurun_out/prof_tb_M1_${TAG} -f python -c "
import ibm_inputs as I, paper_2402_17337_b200 as P
cfg = I.cfg3(1, maxit_p=300)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs()); g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, 0.01)); g.step(1)
" > gpurun_out/ncu_tb_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_tb_${TAG}.log
if [ -n "$BENCH" ]; then
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g clocks %s' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))"
fi
