mkdir -p gpurun_out/r2i
rm -f gpurun_out/r2i/*.log
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2i/bicg_npw1.log 2>&1
BBML_F64_SHORT_NPW=4 timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2i/bicg_npw4.log 2>&1
for q in 1 0; do for npw in 1 2; do
  echo "== QUEUE=$q SHORT_NPW=$npw" >> gpurun_out/r2i/ab.log
  BBML_LM_QUEUE=$q BBML_F64_SHORT_NPW=$npw PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2i/ab.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2i/pytest.log 2>&1; echo pytest=$?
