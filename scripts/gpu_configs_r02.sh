# per-config bench lines (evals/s + e2e), and time-to-best with and without transpositions (R24)
for c in gpt24 unet gns16 llama80; do
  timeout 600 python bench.py --config $c --no-search --no-cpu-baseline --no-variants > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
done
for tp in 0 1; do for c in gpt24 llama80 unet; do
  timeout 900 python bench.py --config $c --transpositions $tp --no-cpu-baseline --no-variants --ttb-configs "" --steps 5 > gpurun_out/ttb_${c}_$tp.json 2> gpurun_out/ttb_${c}_$tp.err; echo "ttb $c tp=$tp rc=$?"
done; done
