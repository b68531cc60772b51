python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
A="--steps 1000 --no-orderings --no-e2e --no-cpu --no-heun --no-orders"
for cfg in "1 256" "0 256" "0 192" "0 128" "1 192"; do
  set -- $cfg
  SEM_K7_WIN=$1 SEM_CHUNK=$2 timeout 600 python bench.py $A > gpurun_out/k7w_w$1_b$2.json 2>gpurun_out/k7w_w$1_b$2.err; echo "w$1 b$2 rc=$?"
done
SEM_K7_WIN=0 SEM_CHUNK=192 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_full or random_state or reduced" > gpurun_out/pytest_w0.log 2>&1; echo "w0 tests rc=$?"
