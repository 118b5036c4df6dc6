"""Model texts for the benchmark configurations.

double_integrator / goddard / quadrotor are the reference's embedded models
(/root/reference/proj/src/bench/problems.cpp:24-95) — model data, reproduced so
that both sides transcribe the identical text. hang_glider / shuttle /
cart_pendulum are the SURVEY.md Appendix B texts (new model data; parity for
them is pinned by running the reference CPU code on the same text).
"""

DOUBLE_INTEGRATOR = """# double integrator, minimum control energy
t in [0, 1], time
x in R^2, state
u in R, control

x(0) == [-1, 0]
x(1) == [0, 0]

derivative(x1)(t) == x2(t)
derivative(x2)(t) == u(t)

integral( 0.5u(t)^2 ) => min
"""

GODDARD = """# Goddard rocket, maximum final altitude
r0 = 1.0
v0 = 0.0
m0 = 1.0
vmax = 0.1
mf = 0.6
Cd = 310.0
Tmax = 3.5
beta = 500.0
b = 2.0

tf in R, variable
t in [0, tf], time
x = (r, v, m) in R^3, state
u in R, control

x(0) == [r0, v0, m0]
m(tf) == mf
0 <= u(t) <= 1
r(t) >= r0
0 <= v(t) <= vmax

derivative(r)(t) == v(t)
derivative(v)(t) == -Cd * v(t)^2 * exp(-beta * (r(t) - 1)) / m(t) - 1 / r(t)^2 + u(t) * Tmax / m(t)
derivative(m)(t) == -b * Tmax * u(t)

r(tf) => max
"""

QUADROTOR = """# quadrotor, reference tracking
T = 1
g = 9.8
r = 0.1

t in [0, T], time
x in R^9, state
u in R^4, control

x(0) == zeros(9)

derivative(x1)(t) == x2(t)
derivative(x2)(t) == u1(t) * cos(x7(t)) * sin(x8(t)) * cos(x9(t)) + u1(t) * sin(x7(t)) * sin(x9(t))
derivative(x3)(t) == x4(t)
derivative(x4)(t) == u1(t) * cos(x7(t)) * sin(x8(t)) * sin(x9(t)) - u1(t) * sin(x7(t)) * cos(x9(t))
derivative(x5)(t) == x6(t)
derivative(x6)(t) == u1(t) * cos(x7(t)) * cos(x8(t)) - g
derivative(x7)(t) == u2(t) * cos(x7(t)) / cos(x8(t)) + u3(t) * sin(x7(t)) / cos(x8(t))
derivative(x8)(t) == -u2(t) * sin(x7(t)) + u3(t) * cos(x7(t))
derivative(x9)(t) == u2(t) * cos(x7(t)) * tan(x8(t)) + u3(t) * sin(x7(t)) * tan(x8(t)) + u4(t)

dt1 = sin(2pi * t / T)
dt3 = 2sin(4pi * t / T)
dt5 = 2t / T

0.5integral( (x1(t) - dt1)^2 + (x3(t) - dt3)^2 + (x5(t) - dt5)^2 + x7(t)^2 + x8(t)^2 + x9(t)^2 + r * (u1(t)^2 + u2(t)^2 + u3(t)^2 + u4(t)^2) ) => min
"""

HANG_GLIDER = """# hang glider (COPS)
um = 2.5
R = 100
C0 = 0.034
k = 0.069662
mass = 100
S = 14
rho = 1.13
g = 9.81
tf in R, variable
t in [0, tf], time
s = (x, y, vx, vy) in R^4, state
cL in R, control
s(0) == [0, 1000, 13.2275675, -1.28750052]
y(tf) == 900
vx(tf) == 13.2275675
vy(tf) == -1.28750052
tf >= 0.1
0 <= cL(t) <= 1.4
x(t) >= 0
vx(t) >= 0
X = (x(t) / R - 2.5)^2
ua = um * (1 - X) * exp(-X)
Vy = vy(t) - ua
vr = sqrt(vx(t)^2 + Vy^2)
D = 0.5 * (C0 + k * cL(t)^2) * rho * S * vr^2
L = 0.5 * cL(t) * rho * S * vr^2
derivative(x)(t) == vx(t)
derivative(y)(t) == vy(t)
derivative(vx)(t) == (-L * Vy / vr - D * vx(t) / vr) / mass
derivative(vy)(t) == (L * vx(t) / vr - D * Vy / vr - mass * g) / mass
x(tf) => max
"""

SHUTTLE = """# space shuttle reentry (Betts ex. 6.1), h in 1e5 ft, v in 1e4 ft/s
w = 203000
g0 = 32.174
mass = w / g0
rho0 = 0.002378
hr = 23800
Re = 20902900
mu = 0.14076539e17
S = 2690
a0 = -0.20704
a1 = 0.029244
b0 = 0.07854
b1 = -0.61592e-2
b2 = 0.621408e-3
tf in R, variable
t in [0, tf], time
s = (h, phi, theta, v, gam, psi) in R^6, state
c = (alpha, beta) in R^2, control
s(0) == [2.6, 0, 0, 2.56, -0.017453292519943295, 1.5707963267948966]
h(tf) == 0.8
v(tf) == 0.25
gam(tf) == -0.08726646259971647
tf >= 100
ah = alpha(t) * 57.29577951308232
CL = a0 + a1 * ah
CD = b0 + b1 * ah + b2 * ah^2
rho = rho0 * exp(-h(t) * 1e5 / hr)
D = 0.5 * CD * S * rho * (v(t) * 1e4)^2
L = 0.5 * CL * S * rho * (v(t) * 1e4)^2
r = Re + h(t) * 1e5
grav = mu / r^2
derivative(h)(t) == v(t) * 1e4 * sin(gam(t)) / 1e5
derivative(phi)(t) == v(t) * 1e4 / r * cos(gam(t)) * sin(psi(t)) / cos(theta(t))
derivative(theta)(t) == v(t) * 1e4 / r * cos(gam(t)) * cos(psi(t))
derivative(v)(t) == (-D / mass - grav * sin(gam(t))) / 1e4
derivative(gam)(t) == L / (mass * v(t) * 1e4) * cos(beta(t)) + cos(gam(t)) * (v(t) * 1e4 / r - grav / (v(t) * 1e4))
derivative(psi)(t) == L * sin(beta(t)) / (mass * v(t) * 1e4 * cos(gam(t))) + v(t) * 1e4 / (r * cos(theta(t))) * cos(gam(t)) * sin(psi(t)) * sin(theta(t))
theta(tf) => max
"""

CART_PENDULUM = """# cart-pendulum swing-up
M = 1
mp = 0.3
l = 0.5
g = 9.81
t in [0, 2], time
s = (p, th, pd, thd) in R^4, state
F in R, control
s(0) == [0, 0, 0, 0]
s(2) == [1, 3.141592653589793, 0, 0]
-20 <= F(t) <= 20
den = M + mp * sin(th(t))^2
derivative(p)(t) == pd(t)
derivative(th)(t) == thd(t)
derivative(pd)(t) == (F(t) + mp * sin(th(t)) * (l * thd(t)^2 + g * cos(th(t)))) / den
derivative(thd)(t) == -(F(t) * cos(th(t)) + mp * l * thd(t)^2 * cos(th(t)) * sin(th(t)) + (M + mp) * g * sin(th(t))) / (l * den)
integral( F(t)^2 ) => min
"""

MODELS = {
    "double_integrator": DOUBLE_INTEGRATOR,
    "goddard": GODDARD,
    "quadrotor": QUADROTOR,
    "hang_glider": HANG_GLIDER,
    "shuttle": SHUTTLE,
    "cart_pendulum": CART_PENDULUM,
}


def cart_pendulum_instance(b: int, batch: int = 4096) -> str:
    """Batch config instance b: terminal target p(2) = 1 + b/batch."""
    target = 1.0 + b / batch
    return CART_PENDULUM.replace("s(2) == [1, 3.141592653589793, 0, 0]",
                                 f"s(2) == [{target!r}, 3.141592653589793, 0, 0]")
