# A/B of an environment switch (run under gpurun): parity subset with the default, then per-op
# timings with VAR=a and VAR=b.  usage: bash tools/gpu_ab_env.sh TAG VAR "a b" "pytest -k" "C5 shell 16" ...
tag=$1; var=$2; vals=$3; kexpr=$4; shift 4
work=("$@")
timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for v in $vals; do
  for a in "${work[@]}"; do env $var=$v timeout 300 python tools/time_op.py $a 3; done > gpurun_out/${tag}_${v}_times.log 2>&1
done
echo done
