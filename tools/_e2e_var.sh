O=gpurun_out/s3_e2evar; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for k in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > $O/b$k.json 2>$O/b$k.err; done
timeout 300 python bench.py > $O/bfull.json 2>$O/bfull.err
tail -2 $O/pytest_gpu.log
for f in b1 b2 b3 bfull; do python -c "import json; d=json.load(open('$O/$f.json')); print('$f', d['ms_per_step'], d['phases_ms_per_step'], d['e2e']['ms_per_step'])"; done
