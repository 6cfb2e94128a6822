mkdir -p gpurun_out/r2s; rm -f gpurun_out/r2s/*
O=gpurun_out/r2s
for prec in 64 32; do
  timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/prof.py --workload app20 --precision $prec --epochs 20 --br-epochs 50 --reps 1 > $O/memcheck_app20_fp$prec.log 2>&1; echo memcheck$prec=$?
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/prof.py --workload suite16 --precision 64 --epochs 3 --br-epochs 20 --reps 1 --app pathfinder,gramschmit,atax > $O/memcheck_suite16_sub.log 2>&1; echo memcheck_suite=$?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 python tools/prof.py --workload app20 --precision 64 --epochs 5 --br-epochs 20 --reps 1 > $O/racecheck_app20.log 2>&1; echo racecheck=$?
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/prof.py --workload app20 --precision 64 --epochs 5 --br-epochs 20 --reps 1 > $O/synccheck_app20.log 2>&1; echo synccheck=$?
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/prof.py --workload wide --kind br --restarts 1 --br-epochs 3 --reps 1 > $O/memcheck_wide.log 2>&1; echo memcheck_wide=$?
tail -3 $O/*.log
