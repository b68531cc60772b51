A="--steps 1000 --no-orderings --no-e2e --no-cpu --no-orders"
for i in 1 2 3; do for v in libsem.so libsem_alt.so; do SEM_LIB=$PWD/paper_2104_08416_b200/$v timeout 900 python bench.py $A > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; h=d['heun']; print('$v leap %.4f k7 %.4f k8 %.4f heun %.4f'%(d['ms_per_step'], r['avg_launch_ms'], r['k8_avg_launch_ms'], h['ms_per_step']))"; done; done
