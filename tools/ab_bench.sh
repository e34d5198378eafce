# Dev tool: short c2 bench lines (uint16 and uint32 residues) -> gpurun_out/ab_*.json
python bench.py --no-cpu --no-check --no-compare > gpurun_out/ab_u16.json 2> gpurun_out/ab.err
python bench.py --no-cpu --no-check --no-compare --io u32 > gpurun_out/ab_u32.json 2>> gpurun_out/ab.err
tail -3 gpurun_out/ab.err
