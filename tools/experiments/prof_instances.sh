for cfg in "K4V2:--kb 4 --vb 2" "K2V2:--kb 2 --vb 2" "K4V4:--kb 4 --vb 4" "K8V4:--kb 8 --vb 4"; do
  name=${cfg%%:*}; args=${cfg#*:}
  bash tools/gpu_prof.sh fin_$name "$args"
done
