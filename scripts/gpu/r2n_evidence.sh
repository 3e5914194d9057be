# round-2 evidence (r02n): smoke, GPU suite, default bench line, reference arm, cfg3 line, launch list,
# ncu of the four cfg4 kernels
TAG=${TAG:-r02n}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${TAG}_pytest.log
timeout 400 python bench.py > gpurun_out/${TAG}_b4.json 2> gpurun_out/${TAG}_b4.err
timeout 300 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b3.json 2> gpurun_out/${TAG}_b3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 2 --profile-run > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k 'regex:fd_tc|gram_tc2|solve_mw|precode_tc2' -s 8 -c 4 -o gpurun_out/${TAG}_cfg4 python bench.py --steps 2 --warmup 2 --profile-run > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b2.json 2> gpurun_out/${TAG}_b2.err
