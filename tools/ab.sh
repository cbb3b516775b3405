# A/B timing of library builds on the bench workload (diagnostic).
# usage: bash tools/ab.sh "label|ENV=..|dir" ...   ms_per_step per config, 2 interleaved rounds
for rep in 1 2; do
for spec in "$@"; do
  label=${spec%%|*}; rest=${spec#*|}; envs=${rest%%|*}; dir=${rest#*|}
  flags="--no-cpu-baseline --no-batched"
  grep -q no-roofline $dir/bench.py && flags="$flags --no-roofline"
  r=$(cd $dir && env $envs python bench.py $flags 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>/dev/null)
  echo "$label $r"
done; done
