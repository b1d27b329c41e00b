for v in "JT_AB=0" "JT_SPLIT_CPASS=0"; do
  echo "[$v]" >> gpurun_out/c4m_ab.txt
  env $v timeout 300 python -c "
import bench, json
print(json.dumps({k:v['cases_per_s'] for k,v in bench.batch_table(configs=('c4M','c2')).items()}))" >> gpurun_out/c4m_ab.txt 2>&1
done
