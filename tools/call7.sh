for pol in "4:24" "4:20" "4:16"; do
  VSDOCK_POLICY=$pol ATOMS=20,32 TAG=c32_$pol timeout 120 python tools/dock_time.py 200000 1 1
  VSDOCK_POLICY=$pol ATOMS=33,64 TAG=c64_$pol timeout 120 python tools/dock_time.py 200000 1 1
  VSDOCK_POLICY=$pol ATOMS=65,96 TAG=c96_$pol timeout 120 python tools/dock_time.py 200000 1 1
done
