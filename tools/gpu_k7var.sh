python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
A="--steps 1000 --no-orderings --no-e2e --no-cpu --no-heun --no-orders"
for cfg in "1 256" "2 256" "2 192" "1 192" "2 128"; do
  set -- $cfg
  SEM_K7_WIN=$1 SEM_CHUNK=$2 timeout 600 python bench.py $A > gpurun_out/k7var_w$1_b$2.json 2>gpurun_out/k7var_w$1_b$2.err; echo "w$1 b$2 rc=$?"
done
SEM_K7_WIN=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_win2.log 2>&1; echo "win2 tests rc=$?"
