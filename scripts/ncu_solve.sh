# ncu --set full of the 5 spectral-solve passes of one 840^3 projection; digests into gpurun_out/$1
O=gpurun_out/${1:-ncu_solve}
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_rfft -s 5 -c 5 -o $O/solve python scripts/ncu_solve.py 840 > $O/solve.log 2>&1
python profiles/ncu_digest.py $O/solve.ncu-rep > $O/solve_digest.txt 2>&1
ncu -i $O/solve.ncu-rep --page raw --csv > $O/solve_raw.csv 2>/dev/null
rm -f $O/solve.ncu-rep
