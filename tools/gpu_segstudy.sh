for cfg in "--rate 500 --delta 0.1 --d1 3.5e-8 --reps 1024" "--rate 500 --delta 1e-5 --d1 3.5e-8 --reps 1024"; do
  tag=$(echo $cfg | tr -d ' -' | tr '.' 'p')
  echo "== $cfg"
  timeout 1200 python -m paper_2504_11320_b200.studies $cfg --out gpurun_out/segstudy_$tag.json
done
