for rep in 1 2 3; do
for cfg in "32 4 1 2" "8 1 1 1" "32 1 1 0" "8 1 0 1"; do
set -- $cfg
python tools/k6_sched.py --reps 60 --warm 10 --mgroup $1 --tps $2 --pola $3 --polb $4 | tail -1
done
done
