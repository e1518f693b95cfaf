rb() { SFB_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
import runpy; m=runpy.run_path('paper_2604_18536_b200/build.py'); m['build'](force=True)"; }
st() { ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_stage" -s 8 -c 8 --csv --log-file gpurun_out/nc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; python profiles/parse_launches.py gpurun_out/nc.csv | head -5; }
rb "-DSFB_STAGE_NOFILL"; st
